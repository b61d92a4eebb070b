# int8 GEMV tests (converter and encoded kernels) + the fp32 bench line (run via gpurun).
mkdir -p gpurun_out
python -m paper_2509_20500_b200.build > /dev/null
timeout 1200 python -m pytest tests/test_i8_gpu.py tests/test_build_plan_gpu.py -q -m gpu -x --durations=5 > gpurun_out/i8_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/i8_tests.log
tail -12 gpurun_out/i8_tests.log
timeout 600 python bench.py --steps 20 --warmup 5 --dtype f32 --no-cpu-baseline > gpurun_out/i8_f32.json 2> gpurun_out/i8_f32.err; echo "bench rc=$?"
python -c "
import json; d=json.load(open('gpurun_out/i8_f32.json')); print(d['value'], d['ms_per_step'], d['roofline']['frac'], d['roofline'].get('kernel')[:20], d['clocks'], d['e2e']['value'], d['gpu_launches'])"
