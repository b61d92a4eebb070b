"""Int8 tensor-core GEMV vs the DMMA / DFMA GEMV on the same plan (GPU scratch check).

python tools/i8_check.py [N] [dtype f32|f64] [V]
Builds P~0 for config 5's flux at N bins, solves V dead times with SPLIDAR_I8=1 and =0 plans and
prints iterations, max |pi_i8 - pi_dmma| (L1 per vector) and the solve time of each.
"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2509_20500_b200 as spl
from workloads import Flux, config

N = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
dt = torch.float32 if (len(sys.argv) < 3 or sys.argv[2] == "f32") else torch.float64
V = int(sys.argv[3]) if len(sys.argv) > 3 else 17
w = config(5)
f0 = w.items[0].flux
f = Flux(f0.t_r, N, f0.tau, f0.sigma, f0.signal, f0.background)
tds = ([w.items[0].t_d] + [it.t_d for it in w.sweep])[:V]
P0 = spl.build_base(f, dt)
torch.cuda.synchronize()
res = {}
for mode in ("1", "0"):
    os.environ["SPLIDAR_I8"] = mode
    plan = spl.Plan(P0, f.t_r, np.array([tds]), tol=1e-12)
    infos = plan.execute(check=False)
    torch.cuda.synchronize()
    ts = []
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        plan.launch()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    res[mode] = (plan.pi[0].detach().cpu().numpy().copy(), [i["iters"] for i in infos],
                 [i["converged"] for i in infos], min(ts))
    plan.close()
pi1, it1, c1, t1 = res["1"]
pi0, it0, c0, t0 = res["0"]
print(f"N={N} {dt} V={V}")
print("iters i8  ", it1, "conv", all(c1))
print("iters dmma", it0, "conv", all(c0))
print("L1(pi_i8 - pi_dmma) per vector max %.3e" % np.max(np.sum(np.abs(pi1 - pi0), axis=1)))
print("solve ms: i8 %.3f  dmma %.3f" % (t1, t0))
