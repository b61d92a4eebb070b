import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import oracle, paper_2509_20500_b200 as spl
from workloads import Flux
f = Flux(100.0, 512, (42.0,), (0.7,), (450.0,), 120.0)
N = 512
P = oracle.build_eq4(f, 0.0)
v = spl.flux_vectors(f)
s = (np.arange(N) + 0.5) * 100 / N
F = np.array([oracle.F(f, t) for t in s]); lam = np.array([oracle.lam(f, t) for t in s]); L = oracle.Lambda(f)
w = lam * np.exp(-F); eL = np.exp(-L)
U = np.cumsum(w[::-1])[::-1]; Lp = np.concatenate([[0], np.cumsum(w)[:-1]]); D = U + eL * Lp
print("Lambda gpu", v["Lambda"].item(), L)
for k, ref in (("F", F), ("lam", lam), ("w", w), ("inv_d", 1 / D)):
    g = v[k].cpu().numpy()
    rel = np.abs(g - ref) / np.abs(ref)
    print(k, "max rel", rel.max(), "at", rel.argmax(), g[rel.argmax()], ref[rel.argmax()])
P0 = spl.build_base(f).cpu().numpy()
err = np.abs(P0 - P)
i = np.unravel_index(err.argmax(), err.shape)
print("P0 max err", err.max(), i, P0[i], P[i], "bad rows", np.where(err.max(1) > 1e-12)[0][:20])
