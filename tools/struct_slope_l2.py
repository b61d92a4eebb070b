"""Per-product cost of the structured lambda_2 kernel: kernel time vs max_iter (scratch)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2509_20500_b200 as spl  # noqa: E402
from workloads import config  # noqa: E402

for k in (3, 4, 5):
    it = config(k).items[0]
    f = it.flux
    shape, S, B = spl.flux_items(f)
    pi, _ = spl.stationary_structured(shape, S, B, [it.t_d])
    res = []
    for n in (4, 8, 16):
        p = spl.StructPlan("lambda2", shape, S, B, [it.t_d], pi=pi, tol=1e-300, max_iter=n)
        ts = []
        for _ in range(5):
            p.launch()
            ts.append(p.info(check=False)[1])
        res.append((n, min(ts)))
        p.close()
    n = np.array([r[0] for r in res], float)
    t = np.array([r[1] for r in res], float)
    a, b = np.polyfit(n, t, 1)
    print(f"lambda2 N={f.n_bins}: " + ", ".join(f"{int(x)}: {y * 1e3:.1f} us" for x, y in res)
          + f" -> {a * 1e3:.2f} us per product + {b * 1e3:.1f} us fixed")
