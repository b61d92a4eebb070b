python __graft_entry__.py > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_structured_gpu.py -q -x 2>&1 | tail -1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launch_struct_c3.csv python bench.py --path structured --workload c3 --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > /dev/null 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_vec --csv --log-file gpurun_out/launch_vec_c5.csv python bench.py --path structured --workload c5 --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > /dev/null 2>&1
grep k_vec gpurun_out/launch_struct_c3.csv | head -1 | awk -F'","' '{print "c3", $5, $NF}'
grep k_vec gpurun_out/launch_vec_c5.csv | head -5 | awk -F'","' '{print "c5", $5, $NF}'
for w in c3 c5; do timeout 300 python bench.py --path structured --workload $w --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('struct $w', round(d['value']), round(d['ms_per_step'],4), round(d['roofline']['kernel_ms_per_step'],4))"; done
