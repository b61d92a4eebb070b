python __graft_entry__.py > gpurun_out/build.log 2>&1
timeout 300 python tools/struct_slope.py 2>&1 | tail -3
timeout 600 python -m pytest tests/test_structured_gpu.py -q -x 2>&1 | tail -1
for w in c5 c4; do timeout 300 python bench.py --path structured --workload $w --no-cpu-baseline > gpurun_out/bench_struct_$w.json 2>/dev/null; python -c "
import json; d=json.load(open('gpurun_out/bench_struct_$w.json')); r=d['roofline']; print('$w', round(d['value']), round(d['ms_per_step'],4), round(r.get('kernel_ms_per_step'),4))"; done
