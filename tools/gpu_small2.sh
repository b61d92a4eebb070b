python __graft_entry__.py > gpurun_out/build.log 2>&1
for w in c1 c2; do timeout 300 python bench.py --workload $w > gpurun_out/bench_$w.json 2> gpurun_out/bench_$w.err; tail -c 600 gpurun_out/bench_$w.err; python -c "
import json; d=json.load(open('gpurun_out/bench_$w.json')); print('$w', d['value'], d['ms_per_step'], d['ms_build_per_step'], d['ms_solve_per_step'], d['e2e']['value'], d['config']['solver'], d['config']['step_as_cuda_graph'], d['gpu_launches'])"; done
timeout 600 python -m pytest tests/test_parity_gpu.py -m gpu -q -x --timeout=300 -k "fused or config1 or config2 or deterministic" 2>&1 | tail -2
