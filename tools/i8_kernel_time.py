"""Per-launch time of the int8 GEMV kernel (eager loop, kineto), for timing experiments.

SPLIDAR_I8_DBG=<bits> python tools/i8_kernel_time.py N f32|f64 V ITERS
(bits: 1 skip the conversion, 2 skip the MMAs; results are then meaningless, only the time counts)
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["SPLIDAR_EAGER"] = "1"
import paper_2509_20500_b200 as spl
from workloads import Flux, config

N = int(sys.argv[1]); dt = torch.float32 if sys.argv[2] == "f32" else torch.float64
V = int(sys.argv[3]); iters = int(sys.argv[4])
w = config(5)
f0 = w.items[0].flux
f = Flux(f0.t_r, N, f0.tau, f0.sigma, f0.signal, f0.background)
tds = ([w.items[0].t_d] + [it.t_d for it in w.sweep])[:V]
P0 = spl.build_base(f, dt)
plan = spl.Plan(P0, f.t_r, np.array([tds]), tol=1e-300, max_iter=iters)
plan.execute(check=False)
torch.cuda.synchronize()
from torch.profiler import profile, ProfilerActivity
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    plan.execute(check=False)
    torch.cuda.synchronize()
ts = {}
for e in prof.events():
    if e.device_type.name == "CUDA":
        nm = e.name
        k = nm[nm.find("k_"):].split("(")[0] if "k_" in nm else nm[:40]
        ts.setdefault(k[:42], []).append(e.device_time if hasattr(e, "device_time") else e.cuda_time)
for k, v in sorted(ts.items(), key=lambda kv: -sum(kv[1])):
    print(f"{k:42s} n={len(v):3d} mean {np.mean(v):9.1f} us  min {np.min(v):9.1f}")
