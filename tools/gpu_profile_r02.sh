#!/bin/bash
# r02 profiling: launch lists of the default (fp64) and fp32 bench commands, one ncu --set full
# capture of each dominant kernel. Every ncu run is after the same command exited 0 without ncu.
mkdir -p gpurun_out
python -m paper_2509_20500_b200.build > /dev/null
export SPLIDAR_EAGER=1      # host loop over the same kernels (ncu does not descend into conditional graph bodies)
for dt in f64 f32; do
  python bench.py --steps 2 --warmup 1 --dtype $dt --no-cpu-baseline --no-e2e > gpurun_out/r02_plain_$dt.json 2>&1 || exit 1
  ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02_launches_c5_$dt.csv \
      python bench.py --steps 2 --warmup 1 --dtype $dt --no-cpu-baseline --no-e2e > gpurun_out/r02_ncu_launch_$dt.log 2>&1
done
ncu --set full --clock-control none --import-source on -k regex:"k_power_step_i8" -s 4 -c 1 -o gpurun_out/r02_full_i8_f32 \
    python bench.py --steps 1 --warmup 1 --dtype f32 --no-cpu-baseline --no-e2e > gpurun_out/r02_ncu_full_i8.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_i8_colexp" -c 1 -o gpurun_out/r02_full_colexp_f32 \
    python bench.py --steps 1 --warmup 1 --dtype f32 --no-cpu-baseline --no-e2e > gpurun_out/r02_ncu_full_colexp.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_power_step<double, 17>|k_power_stepIdLi17" -s 10 -c 1 \
    -o gpurun_out/r02_full_dmma_f64 python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/r02_ncu_full_dmma.log 2>&1
ls -la gpurun_out/r02_*
