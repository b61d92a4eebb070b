"""One structured solve call for ncu (scratch): --case grid256 | c3 | c5."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2509_20500_b200 as spl
from workloads import Flux, config
case = sys.argv[1]
if case.startswith("grid"):
    N = int(case[4:])
    base = Flux(100.0, N, (40.0,), (0.5,), (1.0,), 1.0)
    sv = np.linspace(0.05, 10, 64)
    S, B = np.meshgrid(sv, sv, indexing="ij")
    S = np.tile(S.ravel(), 2); B = np.tile(B.ravel(), 2)
    T = np.repeat([75.0, 95.0], 64 * 64)
    shape = base
elif case == "c4":
    it = config(4).items[0]; shape = it.flux; S = np.ones(1); B = np.array([shape.background]); T = np.array([it.t_d])
elif case == "c3":
    it = config(3).items[0]; shape = it.flux; S = np.ones(1); B = np.array([shape.background]); T = np.array([it.t_d])
else:
    w = config(5); shape = w.items[0].flux
    T = np.array([w.items[0].t_d] + [it.t_d for it in w.sweep]); S = np.ones(17); B = np.full(17, shape.background)
pi, inf = spl.stationary_structured(shape, S, B, T)
if "--l2" in sys.argv:
    spl.second_eigenvalue(shape, S, B, T, pi)
torch.cuda.synchronize()
print(case, sum(i["iters"] for i in inf))
