"""Kernel-level durations (CUPTI via torch.profiler) of the structured calls (scratch)."""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from torch.profiler import profile, ProfilerActivity
import paper_2509_20500_b200 as spl
from workloads import Flux, config

cases = []
w = config(5); f = w.items[0].flux
tds = [w.items[0].t_d] + [it.t_d for it in w.sweep]
cases.append(("c5x17", f, np.ones(17), np.full(17, f.background), np.array(tds)))
it = config(3).items[0]
cases.append(("c3x1", it.flux, np.ones(1), np.array([it.flux.background]), np.array([it.t_d])))
for N in (256, 4096):
    base = Flux(100.0, N, (40.0,), (0.5,), (1.0,), 1.0)
    sv = np.linspace(0.05, 10, 64)
    S, B = np.meshgrid(sv, sv, indexing="ij")
    S = np.tile(S.ravel(), 2); B = np.tile(B.ravel(), 2)
    T = np.repeat([75.0, 95.0], 64 * 64)
    cases.append((f"grid{N}", base, S, B, T))
for name, shape, S, B, T in cases:
    ws = spl.structured_workspace(shape.n_bins, len(set(zip(S, B))), S.size)
    pi, inf = spl.stationary_structured(shape, S, B, T, ws=ws)
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
        pi, inf = spl.stationary_structured(shape, S, B, T, ws=ws)
        l2 = spl.second_eigenvalue(shape, S, B, T, pi, ws=ws)
        torch.cuda.synchronize()
    its = sum(i["iters"] for i in inf)
    l2its = sum(i["iters"] for i in l2)
    ev = [e for e in prof.events() if e.device_type.name == "CUDA"]
    agg = {}
    for e in ev:
        agg.setdefault(e.name[:60], [0, 0.0])
        agg[e.name[:60]][0] += 1
        agg[e.name[:60]][1] += e.device_time_total if hasattr(e, "device_time_total") else e.cuda_time_total
    print(name, "N", shape.n_bins, "items", S.size, "products", its, "l2 products", l2its)
    for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"   {t:10.1f} us  x{n}  {k}")
