"""One dense lambda_2 at config 5 (for ncu / launch lists)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2509_20500_b200 as spl  # noqa: E402
from workloads import config  # noqa: E402

it = config(5).items[0]
f = it.flux
P0 = spl.build_base(f, torch.float64)
pi, _ = spl.stationary(P0, f.t_r, it.t_d)
print(spl.second_eigenvalue_dense(P0, f.t_r, it.t_d, pi))
