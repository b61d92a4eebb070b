python __graft_entry__.py > gpurun_out/build.log 2>&1
python __graft_entry__.py --smoke 2>&1 | tail -1 | cut -c1-120
timeout 1500 python -m pytest tests -m gpu -q -x --timeout=400 > gpurun_out/pytest_gpu.log 2>&1; tail -2 gpurun_out/pytest_gpu.log
for w in c5 c4 c3; do timeout 600 python bench.py --workload $w --no-cpu-baseline > gpurun_out/bench_$w.json 2> gpurun_out/bench_$w.err; tail -c 300 gpurun_out/bench_$w.err; python -c "
import json; d=json.load(open('gpurun_out/bench_$w.json')); r=d['roofline']; print('$w', round(d['value'],1), round(d['ms_per_step'],3), round(d['ms_solve_per_step'],3), round(r['frac'],3), d['iterations'][0][:6])"; done
