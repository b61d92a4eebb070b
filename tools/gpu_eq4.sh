python __graft_entry__.py > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_eq4_gpu.py -m gpu -q --timeout=240 > gpurun_out/pytest_eq4.log 2>&1; tail -5 gpurun_out/pytest_eq4.log
cat > /tmp/eq4_one.py <<'PY'
import sys; sys.path.insert(0, '.')
import torch, paper_2509_20500_b200 as spl
from workloads import config
it = config(5).items[0]
P = spl.build_eq4(it.flux, it.t_d); torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(); spl.build_eq4(it.flux, it.t_d, out=P); e1.record(); torch.cuda.synchronize()
print("eq4 c5 ms", e0.elapsed_time(e1), "entries/s", 32768**2 / e0.elapsed_time(e1) * 1e3)
PY
python /tmp/eq4_one.py
ncu --set full --import-source on --clock-control none -k regex:k_build_eq4 -c 1 -o gpurun_out/ncu_eq4_c5 python /tmp/eq4_one.py > gpurun_out/ncu_eq4.log 2>&1; tail -2 gpurun_out/ncu_eq4.log
