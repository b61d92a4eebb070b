python __graft_entry__.py > gpurun_out/build.log 2>&1
python __graft_entry__.py --smoke 2>&1 | tail -1
timeout 1200 python -m pytest tests/test_parity_gpu.py -m gpu -q -x --timeout=300 > gpurun_out/pytest_parity.log 2>&1; tail -15 gpurun_out/pytest_parity.log
for w in c1 c2; do timeout 300 python bench.py --workload $w --no-cpu-baseline > gpurun_out/bench_$w.json 2> gpurun_out/bench_$w.err; tail -c 300 gpurun_out/bench_$w.err; head -c 250 gpurun_out/bench_$w.json; echo; done
