python __graft_entry__.py > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_structured_gpu.py -m gpu -q --timeout=240 > gpurun_out/pytest_struct.log 2>&1; tail -2 gpurun_out/pytest_struct.log
for w in c5 c3 grid c4; do timeout 300 python bench.py --path structured --workload $w > gpurun_out/bench_struct_$w.json 2> gpurun_out/bench_struct_$w.err; tail -c 400 gpurun_out/bench_struct_$w.err; done
for w in grid c5 c1; do timeout 300 python bench.py --path spectral --workload $w > gpurun_out/bench_spec_$w.json 2> gpurun_out/bench_spec_$w.err; tail -c 400 gpurun_out/bench_spec_$w.err; done
for f in gpurun_out/bench_struct_*.json gpurun_out/bench_spec_*.json; do echo $f; python -c "
import json,sys; d=json.load(open('$f')); r=d['roofline']; print(d['value'], d['unit'], 'ms/step', round(d['ms_per_step'],3), 'kernel ms', round(r['kernel_ms_per_step'],3), 'TF', round(r['achieved'],3), 'frac', round(r['frac'],4), 'e2e', d['e2e']['value'] if d['e2e'] else None, 'cpu', d.get('cpu_baseline',{}) and d['cpu_baseline']['value'], d['converged'])"; done
