set -x
python __graft_entry__.py > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_structured_gpu.py -m gpu -q --timeout=240 > gpurun_out/pytest_struct.log 2>&1; tail -5 gpurun_out/pytest_struct.log
timeout 600 python tools/struct_perf.py > gpurun_out/struct_perf.log 2>&1; cat gpurun_out/struct_perf.log
