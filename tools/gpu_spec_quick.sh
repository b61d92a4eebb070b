python __graft_entry__.py > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_structured_gpu.py -m gpu -q --timeout=240 -x > gpurun_out/pytest_struct.log 2>&1; tail -2 gpurun_out/pytest_struct.log
python tools/struct_prof.py 2>&1 | grep -v Warning | grep -E "^[a-z]|k_struct_lambda2"
for w in grid c5; do timeout 300 python bench.py --path spectral --workload $w --no-cpu-baseline > gpurun_out/bench_spec_$w.json 2>/dev/null; python -c "
import json; d=json.load(open('gpurun_out/bench_spec_$w.json')); r=d['roofline']; print('$w', round(d['value']), d['ms_per_step'], r['kernel_ms_per_step'], round(r['frac'],4))"; done
