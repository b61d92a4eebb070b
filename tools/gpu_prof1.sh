python __graft_entry__.py > gpurun_out/build.log 2>&1
timeout 300 python -m pytest tests/test_parity_gpu.py -q -x --timeout=120 -k "tiny" 2>&1 | tail -3
CMD="python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline"
SPLIDAR_EAGER=1 $CMD > gpurun_out/plain.log 2>&1 && \
SPLIDAR_EAGER=1 ncu --set full --clock-control none --import-source on -k regex:k_power_step -s 10 -c 1 -o gpurun_out/prof_step_nv1 $CMD > gpurun_out/ncu1.log 2>&1; \
SPLIDAR_EAGER=1 ncu --set full --clock-control none --import-source on -k regex:k_power_step -s 30 -c 1 -o gpurun_out/prof_step_nv16 $CMD > gpurun_out/ncu2.log 2>&1; \
SPLIDAR_EAGER=1 ncu --set full --clock-control none --import-source on -k regex:k_build -c 1 -o gpurun_out/prof_build $CMD > gpurun_out/ncu3.log 2>&1
ls -la gpurun_out
