python __graft_entry__.py > gpurun_out/build.log 2>&1
python __graft_entry__.py --smoke 2>&1 | tail -2
timeout 600 python -m pytest tests/test_parity_gpu.py -q -x --timeout=120 -k "stationary or plan or config or tiny or constant or determ or noconv or flux_vectors" 2>&1 | tail -5
python bench.py --no-cpu-baseline > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err; echo c5 rc=$?
for w in c3 c4; do python bench.py --workload $w --no-cpu-baseline > gpurun_out/bench_$w.json 2>gpurun_out/bench_$w.err; done
python bench.py --dtype f32 --no-cpu-baseline > gpurun_out/bench_c5_f32.json 2>&1
SPLIDAR_EAGER=1 python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/plain.log 2>&1 && \
SPLIDAR_EAGER=1 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c5.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ncu.log 2>&1
echo done
