# structured / spectral: parity tests, per-product slopes, bench lines
python __graft_entry__.py > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_structured_gpu.py tests/test_cli.py -q -x 2>&1 | tail -1
timeout 300 python tools/struct_slope_l2.py 2>&1 | grep lambda2
timeout 300 python tools/struct_slope.py 2>&1 | grep "N="
for w in c5 c3 c4 grid; do timeout 300 python bench.py --path structured --workload $w --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('struct $w', round(d['value']), round(d['ms_per_step'],4), round(d['roofline']['kernel_ms_per_step'],4))"; done
for w in c5 c4 c1 grid; do timeout 300 python bench.py --path spectral --workload $w --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('spec $w', round(d['value']), round(d['ms_per_step'],4), round(d['roofline']['kernel_ms_per_step'],4))"; done
