python __graft_entry__.py > gpurun_out/build.log 2>&1
timeout 600 python -m pytest tests/test_structured_gpu.py -q -x -k "lambda2 or mixing or traj" 2>&1 | tail -1
for w in c5 c4 grid; do timeout 300 python bench.py --path spectral --workload $w --no-cpu-baseline > gpurun_out/bench_spec_$w.json 2>/dev/null; python -c "
import json; d=json.load(open('gpurun_out/bench_spec_$w.json')); r=d['roofline']; print('spec $w', round(d['value']), round(d['ms_per_step'],4), round(r.get('kernel_ms_per_step', 0) or 0,4))"; done
