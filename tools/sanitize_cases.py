"""Small instances of every kernel family, for compute-sanitizer (memcheck / synccheck / initcheck /
racecheck): python tools/sanitize_cases.py. Prints one line per case; exits 1 on a wrong result."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2509_20500_b200 as spl
from paper_2509_20500_b200.shard import row_block
from workloads import Flux, config, random_flux

ok = True


def report(name, cond):
    global ok
    ok &= bool(cond)
    print(f"{name}: {'ok' if cond else 'FAIL'}", flush=True)


rng = np.random.default_rng(3)
# c1: fused small-N solver, flux vectors (k_vec_small), build, apply_deadtime, eq4
it = config(1).items[0]
f = it.flux
P0 = spl.build_base(f, torch.float64)
P = spl.apply_deadtime(P0, f.t_r, it.t_d)
pi, info = spl.stationary(P0, f.t_r, it.t_d)
E4 = spl.build_eq4(f, it.t_d)
report("c1 fused + build + deadtime + eq4", info["converged"] and float((P - E4).abs().max()) < 1e-12)
# graph path (conditional WHILE), DMMA V = 8 and 32, N = 3000 (ragged strips)
g = random_flux(rng, 3000, 2, s_range=(0.5, 2), b_range=(0.2, 1))
P0g = spl.build_base(g, torch.float64)
for V in (8, 32):
    os.environ["SPLIDAR_FUSED"] = "0"
    plan = spl.Plan(P0g, g.t_r, np.array([rng.uniform(0, 300, V)]), tol=1e-12)
    inf = plan.execute()
    report(f"graph path N=3000 V={V}", all(i["converged"] for i in inf))
    plan.close()
# tiled flux vectors (N = 9001) and a 1-vector solve
h = random_flux(rng, 9001, 1, s_range=(0.5, 2), b_range=(0.2, 1))
P0h = spl.build_base(h, torch.float32)
pih, infh = spl.stationary(P0h, h.t_r, 123.0)
report("N=9001 fp32 tiled vectors + DFMA GEMV", infh["converged"])
del P0h
# int8 tensor-core GEMV (fp32, V = 17), N = 4096
f5 = config(5).items[0].flux
q = Flux(f5.t_r, 4096, f5.tau, f5.sigma, f5.signal, f5.background)
P0q = spl.build_base(q, torch.float32)
plan = spl.Plan(P0q, q.t_r, np.array([np.linspace(10, 500, 17)]), tol=1e-12)
inf = plan.execute()
report("int8 tensor-core GEMV N=4096 V=17", plan.gemv() == "tensor_i8" and all(i["converged"] for i in inf))
plan.close()
# row shards (2 simulated ranks)
plans = []
for r in range(2):
    r0, n = row_block(4096, r, 2)
    plans.append(spl.ShardPlan(spl.build_base_rows(q, r0, n, torch.float64), r0, 4096, q.t_r, [50.0, 430.0]))
for p in plans:
    p.init()
while True:
    for p in plans:
        p.gemv()
    s = plans[0].ypart + plans[1].ypart
    for p in plans:
        p.ypart.copy_(s)
    if not all([p.check() for p in plans]):
        break
report("row shards", all(i["converged"] for i in plans[0].finish()))
# structured teams: warp (256), CTA (4096), cluster (12289: a 1-position CTA), lambda_2, mixing, trajectory
for N in (256, 4096, 12289):
    ff = Flux(100.0, N, (40.0,), (0.5,), (1.0,), 0.5)
    shape, S, B = spl.flux_items(ff)
    pis, infs = spl.stationary_structured(shape, S, B, [75.0])
    l2 = spl.second_eigenvalue(shape, S, B, [75.0], pis)[0]
    report(f"structured + lambda2 N={N}", infs[0]["converged"] and 0 < l2["modulus"] < 1)
ff = Flux(100.0, 256, (40.0,), (0.5,), (1.0,), 0.5)
pis, _ = spl.stationary_structured(*spl.flux_items(ff), [75.0])
ms = spl.mixing_steps(ff, 75.0, pis[0])
tr = spl.bin_trajectory(ff, 75.0, pis[0], 10, 20)
report("mixing + trajectory", ms is not None and tr is not None)
# lambda_2 of a stored matrix (graph: GEMV + dots + update)
l2d = spl.second_eigenvalue_dense(P0, f.t_r, it.t_d, pi)
report("lambda2 dense", l2d["converged"])
# Monte Carlo
shape, S, B = spl.flux_items(f)
hist, qr, tr2 = spl.monte_carlo(shape, S, B, [it.t_d], 7, 4, 16, n_burn=10, n_regs=2000, n_record=8)
report("monte carlo", int(hist.sum()) > 0)
torch.cuda.synchronize()
sys.exit(0 if ok else 1)
