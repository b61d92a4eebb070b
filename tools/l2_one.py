"""One structured lambda_2 solve of config k's first item (for ncu): python tools/l2_one.py 5"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2509_20500_b200 as spl  # noqa: E402
from workloads import config  # noqa: E402

it = config(int(sys.argv[1])).items[0]
shape, S, B = spl.flux_items(it.flux)
pi, _ = spl.stationary_structured(shape, S, B, [it.t_d])
print(spl.second_eigenvalue(shape, S, B, [it.t_d], pi)[0])
