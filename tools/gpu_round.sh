#!/bin/bash
# Full GPU check: tests, smoke, default bench line, fp32 bench line.
mkdir -p gpurun_out
python -m paper_2509_20500_b200.build > /dev/null
python -m pytest tests -m gpu -x -q --durations=10 > gpurun_out/gputest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gputest.log
python __graft_entry__.py --smoke > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
python bench.py --steps 20 --warmup 5 > gpurun_out/bench_c5_f64.json 2> gpurun_out/bench_c5_f64.err
python bench.py --steps 20 --warmup 5 --dtype f32 --no-cpu-baseline > gpurun_out/bench_c5_f32.json 2> gpurun_out/bench_c5_f32.err
tail -3 gpurun_out/gputest.log; tail -2 gpurun_out/smoke.log
for f in gpurun_out/bench_c5_f64.json gpurun_out/bench_c5_f32.json; do python -c "
import json,sys; d=json.load(open('$f')); print('$f', round(d['value'],1), round(d['ms_per_step'],2), d['roofline']['kernel'][:30], round(d['roofline']['frac'],3), d['clocks'], d['e2e']['value'] if d.get('e2e') else None)"; done
