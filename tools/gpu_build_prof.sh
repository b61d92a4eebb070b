#!/bin/bash
# Build-phase kernels of the fp32 (encoded) and fp64 c5 commands: launch list and one ncu --set full
# capture of k_build each, after the same command exited 0 without ncu (run via gpurun).
mkdir -p gpurun_out
export SPLIDAR_EAGER=1
python bench.py --steps 1 --warmup 1 --dtype f32 --no-cpu-baseline --no-e2e > gpurun_out/bp_plain.json 2>&1 || exit 1
ncu --set full --clock-control none --import-source on -k regex:"k_build" -c 1 -o gpurun_out/bp_full_f32 \
    python bench.py --steps 1 --warmup 1 --dtype f32 --no-cpu-baseline --no-e2e > gpurun_out/bp_ncu_f32.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_build" -c 1 -o gpurun_out/bp_full_f64 \
    python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/bp_ncu_f64.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/bp_launches_f32.csv \
    python bench.py --steps 1 --warmup 1 --dtype f32 --no-cpu-baseline --no-e2e > gpurun_out/bp_ncu_launch.log 2>&1
ls -la gpurun_out/bp_*
