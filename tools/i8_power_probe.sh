# Sustained-load probe: per-pass GEMV time, SM clock and board power for the c5 17-vector pass on the
# DMMA kernel and the int8 kernel (fp32 / fp64 storage), with and without the converters
# (SPLIDAR_I8_DBG=1: conversion skipped, results meaningless). Run via gpurun from the repo root.
O=gpurun_out; mkdir -p $O
python -m paper_2509_20500_b200.build > /dev/null
probe() {
  local name=$1; shift
  nvidia-smi --query-gpu=clocks.sm,power.draw --format=csv,noheader,nounits -lms 100 > $O/pp_$name.smi &
  local sp=$!
  env "$@" python tools/i8_kernel_time.py 32768 $DT 17 $ITERS > $O/pp_$name.txt 2>&1
  kill $sp
  python - "$O/pp_$name.smi" "$O/pp_$name.txt" "$name" <<'PY'
import sys, numpy as np
rows = [l.split(',') for l in open(sys.argv[1]) if l.strip()]
c = np.array([float(r[0]) for r in rows]); p = np.array([float(r[1]) for r in rows])
busy = p > 300
print(sys.argv[3], 'sm_mhz median(load) %.0f' % np.median(c[busy]) if busy.any() else 'idle', 'power max %.0f' % p.max(),
      '|', [l.strip() for l in open(sys.argv[2]) if 'k_power' in l][:2])
PY
}
ITERS=1500
DT=f32 probe f32_i8 SPLIDAR_I8=1
DT=f32 probe f32_i8_noconv SPLIDAR_I8=1 SPLIDAR_I8_DBG=1
DT=f32 probe f32_dmma SPLIDAR_I8=0
ITERS=1000
DT=f64 probe f64_dmma SPLIDAR_I8=0
DT=f64 probe f64_i8 SPLIDAR_I8=2
DT=f64 probe f64_i8_noconv SPLIDAR_I8=2 SPLIDAR_I8_DBG=1
