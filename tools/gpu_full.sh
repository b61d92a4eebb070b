python __graft_entry__.py > gpurun_out/build.log 2>&1
python __graft_entry__.py --smoke 2>&1 | tail -1
timeout 1500 python -m pytest tests -m gpu -q -x --timeout=400 > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
timeout 600 python bench.py > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err; head -c 400 gpurun_out/bench_c5.json
