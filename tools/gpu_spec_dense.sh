# dense lambda_2: timing lines + the eager-mode launch list (kernel shares) at config 5
python __graft_entry__.py > gpurun_out/build.log 2>&1
timeout 300 python tools/spec_dense_time.py > gpurun_out/spec_dense_time.jsonl 2>&1; cat gpurun_out/spec_dense_time.jsonl
cat > /tmp/sd_one.py <<'PY'
import sys, torch
sys.path.insert(0, ".")
import paper_2509_20500_b200 as spl
from workloads import config
it = config(5).items[0]; f = it.flux
P0 = spl.build_base(f, torch.float64)
pi, _ = spl.stationary(P0, f.t_r, it.t_d)
print(spl.second_eigenvalue_dense(P0, f.t_r, it.t_d, pi))
PY
SPLIDAR_EAGER=1 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_spec_dense_c5.csv python /tmp/sd_one.py > gpurun_out/ncu_sd.log 2>&1; tail -2 gpurun_out/ncu_sd.log
