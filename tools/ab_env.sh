#!/bin/bash
# Same-box A/B of one library build under two environment settings (run via gpurun), alternating.
# Usage: bash tools/ab_env.sh REPS "VAR=base_value" "VAR=new_value" "<bench args>"
REPS=$1; A=$2; B=$3; ARGS=$4
mkdir -p gpurun_out
for i in $(seq 1 $REPS); do
  for v in "$A" "$B"; do
    env $v timeout -s KILL 600 python bench.py $ARGS --no-cpu-baseline > gpurun_out/ab_env.json 2> gpurun_out/ab_env.err
    python -c "
import json; d=json.load(open('gpurun_out/ab_env.json')); r=d.get('roofline') or {}
print('$v', round(d['value'],2), 'ms/step', round(d['ms_per_step'],4), 'build', d.get('ms_build_per_step'), 'solve', d.get('ms_solve_per_step'), d['clocks']['sm_mhz'], 'frac', round(r.get('frac') or 0,4), 'e2e', round(d['e2e']['value'],1) if d.get('e2e') else None)"
  done
done
