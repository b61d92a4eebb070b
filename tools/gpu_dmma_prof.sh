#!/bin/bash
mkdir -p gpurun_out
python -m paper_2509_20500_b200.build > /dev/null
SPLIDAR_EAGER=1 ncu --set full --clock-control none --import-source on -k regex:k_power_step -s 10 -c 1 \
    -o gpurun_out/r02_full_dmma_f64 python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/r02_ncu_full_dmma.log 2>&1
SPLIDAR_EAGER=1 ncu --set full --clock-control none --import-source on -k regex:k_power_step_i8 -s 4 -c 1 \
    -o gpurun_out/r02_full_i8_f32b python bench.py --steps 1 --warmup 1 --dtype f32 --no-cpu-baseline --no-e2e > gpurun_out/r02_ncu_full_i8b.log 2>&1
bash tools/gpu_round.sh
