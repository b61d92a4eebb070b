python __graft_entry__.py > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_mc_gpu.py -m gpu -q --timeout=240 > gpurun_out/pytest_mc.log 2>&1; tail -30 gpurun_out/pytest_mc.log
