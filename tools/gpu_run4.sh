set -x
python __graft_entry__.py > gpurun_out/build.log 2>&1
python __graft_entry__.py --smoke 2>&1 | tail -1
timeout 900 python -m pytest tests -m gpu -q -x --timeout=300 > gpurun_out/pytest_gpu.log 2>&1; tail -2 gpurun_out/pytest_gpu.log
python bench.py > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err
for w in c1 c2 c3 c4; do python bench.py --workload $w --no-cpu-baseline > gpurun_out/bench_$w.json 2>gpurun_out/bench_$w.err; done
python bench.py --dtype f32 --no-cpu-baseline > gpurun_out/bench_c5_f32.json 2>&1
python bench.py --mode exp --no-cpu-baseline > gpurun_out/bench_c5_exp.json 2>&1
python bench.py --impl reference --steps 1 > gpurun_out/bench_ref_c5.json 2>&1
echo done
