set -x
python __graft_entry__.py
python bench.py > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err; echo rc=$?
for w in c1 c2 c3 c4; do python bench.py --workload $w --no-cpu-baseline > gpurun_out/bench_$w.json 2>gpurun_out/bench_$w.err; done
python bench.py --dtype f32 --no-cpu-baseline > gpurun_out/bench_c5_f32.json 2>&1
python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c5.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ncu.log 2>&1
echo done
