python __graft_entry__.py > gpurun_out/build.log 2>&1
CMD="python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline"
SPLIDAR_EAGER=1 ncu --set full --import-source on --clock-control none -k regex:k_power_step -s 10 -c 1 -o gpurun_out/ncu_c5_step17 $CMD > gpurun_out/ncu_c5_step17.log 2>&1
SPLIDAR_EAGER=1 ncu --set full --import-source on --clock-control none -k regex:k_build -c 1 -o gpurun_out/ncu_c5_build $CMD > gpurun_out/ncu_c5_build.log 2>&1
ls -la gpurun_out/ncu_c5_*
