#!/bin/bash
# Fused small-N solver (k_power_fused, st.async exchanges) at c1 and c2: one ncu --set full capture
# each, after the same command exited 0 without ncu (run via gpurun).
mkdir -p gpurun_out
for w in c1 c2; do
  python bench.py --workload $w --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/fp_$w.json 2>&1 || exit 1
  SPLIDAR_EAGER=1 timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:"k_power_fused" -c 1 \
      -o gpurun_out/fp_full_$w python bench.py --workload $w --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/fp_ncu_$w.log 2>&1
done
ls -la gpurun_out/fp_*
