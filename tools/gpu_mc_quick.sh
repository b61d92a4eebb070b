python __graft_entry__.py > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_mc_gpu.py -m gpu -q -x --timeout=300 2>&1 | tail -2
for w in grid c1; do timeout 600 python bench.py --path mc --workload $w --steps 3 --warmup 1 --no-cpu-baseline > gpurun_out/bench_mc_$w.json 2>/dev/null; python -c "
import json; d=json.load(open('gpurun_out/bench_mc_$w.json')); print('$w', '%.4g'%d['value'], round(d['ms_per_step'],1))"; done
