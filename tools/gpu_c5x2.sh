python __graft_entry__.py > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_parity_gpu.py -m gpu -q -x --timeout=400 -k "multivector or config5 or stationary or noconv or deterministic" > gpurun_out/pytest_p.log 2>&1; tail -1 gpurun_out/pytest_p.log
for i in 1 2; do for w in c5 c3; do timeout 600 python bench.py --workload $w --no-cpu-baseline --no-e2e > gpurun_out/bench_$w.json 2>/dev/null; python -c "
import json; d=json.load(open('gpurun_out/bench_$w.json')); r=d['roofline']; print('$w', round(d['value'],1), round(d['ms_per_step'],3), round(r['frac'],3), d['clocks']['sm_mhz'])"; done; done
