#!/bin/bash
# ncu --set full of k_power_step<double,17> at three passes of one c5 solve (run via gpurun, after the
# same command exited 0 without ncu): launch 10 (17 vectors running), 27 (7) and 36 (3) of the warm-up
# step -- the DMMA share of the pass falls as converged vectors free their groups.
mkdir -p gpurun_out
SPLIDAR_EAGER=1 python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/dmma_late_plain.json 2> gpurun_out/dmma_late_plain.err || exit 1
for s in 10 27 36; do
    SPLIDAR_EAGER=1 ncu --set full --clock-control none --import-source on -k regex:k_power_step -s $s -c 1 \
        -f -o gpurun_out/r02_dmma_pass$s python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/r02_dmma_pass$s.log 2>&1
    ncu -i gpurun_out/r02_dmma_pass$s.ncu-rep --page raw --csv > gpurun_out/r02_dmma_pass$s.csv 2>/dev/null
done
