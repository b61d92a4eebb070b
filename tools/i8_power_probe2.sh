# Same-box A/B under sustained load (fp64 storage, c5 17-vector pass): DMMA kernel vs the int8 kernel
# without its conversion step (SPLIDAR_I8_DBG=1: the time of an encoded-storage kernel; results
# meaningless), interleaved, 3000 passes each. Run via gpurun from the repo root.
O=gpurun_out; mkdir -p $O
python -m paper_2509_20500_b200.build > /dev/null
probe() {
  local name=$1; shift
  nvidia-smi --query-gpu=clocks.sm,power.draw --format=csv,noheader,nounits -lms 100 > $O/pq_$name.smi &
  local sp=$!
  env "$@" python tools/i8_kernel_time.py 32768 f64 17 3000 > $O/pq_$name.txt 2>&1
  kill $sp
  python - "$O/pq_$name.smi" "$O/pq_$name.txt" "$name" <<'PY'
import sys, numpy as np
rows = [l.split(',') for l in open(sys.argv[1]) if l.strip()]
c = np.array([float(r[0]) for r in rows]); p = np.array([float(r[1]) for r in rows])
busy = p > 300
print(sys.argv[3], 'sm_mhz median(load) %.0f' % np.median(c[busy]) if busy.any() else 'idle', 'power median %.0f' % np.median(p[busy]),
      '|', [l.strip()[:75] for l in open(sys.argv[2]) if 'k_power_step' in l][:2])
PY
}
probe dmma_1 SPLIDAR_I8=0
probe noconv_1 SPLIDAR_I8=2 SPLIDAR_I8_DBG=1
probe dmma_2 SPLIDAR_I8=0
probe noconv_2 SPLIDAR_I8=2 SPLIDAR_I8_DBG=1
probe conv_1 SPLIDAR_I8=2
