python __graft_entry__.py > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_structured_gpu.py -m gpu -q --timeout=240 > gpurun_out/pytest_struct.log 2>&1; tail -3 gpurun_out/pytest_struct.log
python tools/struct_prof.py 2>&1 | grep -v Warning | grep -E "^[a-z]|k_struct"
