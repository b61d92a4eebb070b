#!/bin/bash
# Same-box A/B of two builds of libsplidar.so (run via gpurun): ab/base.so vs ab/new.so, alternating,
# REPS times each, one bench line per run. Usage: bash tools/ab_lib.sh REPS "<bench args>"
REPS=${1:-2}; ARGS=${2:-}
mkdir -p gpurun_out
LIB=paper_2509_20500_b200/lib/libsplidar.so
for i in $(seq 1 $REPS); do
  for v in base new; do
    cp ab/$v.so $LIB && touch $LIB
    timeout -s KILL 600 python bench.py $ARGS --no-cpu-baseline > gpurun_out/ab_$v.json 2> gpurun_out/ab_$v.err
    python -c "
import json; d=json.load(open('gpurun_out/ab_$v.json')); r=d.get('roofline') or {}
print('$v', round(d['value'],2), 'ms/step', round(d['ms_per_step'],4), 'build', d.get('ms_build_per_step'), 'solve', d.get('ms_solve_per_step'), d['clocks']['sm_mhz'], 'frac', round(r.get('frac') or 0,4), 'e2e', round(d['e2e']['value'],1) if d.get('e2e') else None)"
  done
done
cp ab/new.so $LIB && touch $LIB
