#!/bin/bash
# Encoded-storage int8 GEMV (k_power_step_i8e): launch list of the fp32 bench command and one
# ncu --set full capture, each after the same command exited 0 without ncu (run via gpurun).
mkdir -p gpurun_out
python -m paper_2509_20500_b200.build > /dev/null
export SPLIDAR_EAGER=1
python bench.py --steps 2 --warmup 1 --dtype f32 --no-cpu-baseline --no-e2e > gpurun_out/enc_plain.json 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/enc_launches_f32.csv \
    python bench.py --steps 2 --warmup 3 --dtype f32 --no-cpu-baseline --no-e2e > gpurun_out/enc_ncu_launch.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_power_step_i8e" -s 6 -c 1 -o gpurun_out/enc_full_i8e \
    python bench.py --steps 1 --warmup 1 --dtype f32 --no-cpu-baseline --no-e2e > gpurun_out/enc_ncu_full.log 2>&1
ls -la gpurun_out/enc_*
