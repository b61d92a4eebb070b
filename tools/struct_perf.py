"""Times the structured (matrix-free) kernels: per-product latency vs N, and throughput of batched
(S, B) grids (scratch measurement; numbers go to DESIGN.md / profiles)."""
import sys, os, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2509_20500_b200 as spl
from workloads import Flux, config


def timeit(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); fn(); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) / 1e3)
    return min(ts)


out = {}
for k in (1, 2, 3, 4, 5):
    w = config(k)
    f = w.items[0].flux
    tds = [w.items[0].t_d] + [it.t_d for it in w.sweep]
    shape, S, B = spl.flux_items(f)
    S = np.repeat(S, len(tds)); B = np.repeat(B, len(tds))
    ws = spl.structured_workspace(f.n_bins, 1, len(tds))
    res = {}
    def run():
        res["pi"], res["inf"] = spl.stationary_structured(shape, S, B, tds, ws=ws)
    t = timeit(run)
    its = [i["iters"] for i in res["inf"]]
    out[f"c{k}_solve"] = {"N": f.n_bins, "items": len(tds), "s": t, "iters_max": max(its), "iters_sum": sum(its),
                          "us_per_product_max": t / max(its) * 1e6}
    pi = res["pi"]
    def lam():
        res["l2"] = spl.second_eigenvalue(shape, S, B, tds, pi, ws=ws)
    t2 = timeit(lam, 3)
    out[f"c{k}_lambda2"] = {"s": t2, "iters": [i["iters"] for i in res["l2"]],
                            "modulus": [round(i["modulus"], 6) for i in res["l2"]]}
    print(json.dumps({f"c{k}": [out[f"c{k}_solve"], out[f"c{k}_lambda2"]]}), flush=True)

# Fig. 3c / Fig. 4-like grids: S, B in [0.05, 10] (64 x 64), t_d in {75, 95}, N = 256 and 1024
for N in (256, 1024, 4096):
    base = Flux(100.0, N, (40.0,), (0.5,), (1.0,), 1.0)
    sv = np.linspace(0.05, 10, 64)
    S, B = np.meshgrid(sv, sv, indexing="ij")
    S = np.tile(S.ravel(), 2); B = np.tile(B.ravel(), 2)
    T = np.repeat([75.0, 95.0], 64 * 64)
    ws = spl.structured_workspace(N, 64 * 64, S.size)
    res = {}
    def run():
        res["pi"], res["inf"] = spl.stationary_structured(base, S, B, T, ws=ws)
    t = timeit(run, 3)
    its = np.array([i["iters"] for i in res["inf"]])
    def lam():
        res["l2"] = spl.second_eigenvalue(base, S, B, T, res["pi"], ws=ws)
    t2 = timeit(lam, 3)
    l2its = np.array([i["iters"] for i in res["l2"]])
    print(json.dumps({"grid": N, "items": int(S.size), "solve_s": t, "solves_per_s": S.size / t,
                      "iters_sum": int(its.sum()), "elem_products_per_s": float(its.sum()) * N / t,
                      "lambda2_s": t2, "l2_iters_sum": int(l2its.sum()), "l2_iters_max": int(l2its.max()),
                      "l2_conv": int(sum(i["converged"] for i in res["l2"]))}), flush=True)

# mixing steps
for k in (1, 2, 3):
    it = config(k).items[0]
    f = it.flux
    pi, _ = spl.stationary_structured(*spl.flux_items(f), [it.t_d], tol=1e-14)
    res = {}
    def mix():
        res["n"] = spl.mixing_steps(f, it.t_d, pi[0])
    t = timeit(mix, 3)
    print(json.dumps({"mixing": f"c{k}", "N": f.n_bins, "s": t, "n": res["n"][0],
                      "sum_ni": int(res["n"][1].sum())}), flush=True)
