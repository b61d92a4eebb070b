python __graft_entry__.py > gpurun_out/build.log 2>&1
CMD="python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline"
SPLIDAR_EAGER=1 $CMD > gpurun_out/plain.log 2>&1 && \
SPLIDAR_EAGER=1 ncu --set full --clock-control none --import-source on -k regex:k_power_step -s 5 -c 1 -o gpurun_out/prof_nv24_all $CMD > gpurun_out/ncu1.log 2>&1; \
SPLIDAR_EAGER=1 ncu --set full --clock-control none --import-source on -k regex:k_power_step -s 38 -c 1 -o gpurun_out/prof_nv24_one $CMD > gpurun_out/ncu2.log 2>&1
ls gpurun_out
