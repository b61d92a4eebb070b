python __graft_entry__.py > gpurun_out/build.log 2>&1
timeout 1200 python -m pytest tests/test_parity_gpu.py tests/test_cli.py -m gpu -q -x --timeout=400 > gpurun_out/pytest_parity.log 2>&1; tail -2 gpurun_out/pytest_parity.log
for w in c2 c1; do timeout 300 python bench.py --workload $w --no-cpu-baseline > gpurun_out/bench_$w.json 2> gpurun_out/bench_$w.err; tail -c 300 gpurun_out/bench_$w.err; python -c "
import json; d=json.load(open('gpurun_out/bench_$w.json')); print('$w', round(d['value']), d['ms_per_step'], d['ms_build_per_step'], d['ms_solve_per_step'])"; done
