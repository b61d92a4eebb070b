"""Host-side cost of one public one-shot c1 step (build_base + stationary_multi + pi to host)."""
import os, sys, time
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2509_20500_b200 as spl
from workloads import config
it = config(1).items[0]; f = it.flux
P0 = spl.empty_matrix(f.n_bins, torch.float64)
wsb = spl.workspace(f.n_bins)
pi_host = torch.empty((1, f.n_bins), dtype=torch.float64, pin_memory=True)
T = np.array([[it.t_d]])
def one(tim):
    t0 = time.perf_counter(); spl.build_base(f, torch.float64, out=P0, ws=wsb); t1 = time.perf_counter()
    spl.stationary_multi(P0, f.t_r, T, out_host=pi_host); t2 = time.perf_counter(); t3 = t2
    tim.append((t1 - t0, t2 - t1, t3 - t2))
tim = []
for _ in range(50): one(tim)
tim = []
for _ in range(200): one(tim)
a = np.median(np.array(tim), axis=0) * 1e6
print("build %.1f us  stationary %.1f us  copy+sync %.1f us  total %.1f" % (a[0], a[1], a[2], a.sum()))
# pieces of stationary_multi
ws = spl.workspace(f.n_bins, 1, 1); pi = torch.empty((1, 1, f.n_bins), dtype=torch.float64, device="cuda")
ts = []
for _ in range(200):
    t0 = time.perf_counter(); spl.stationary_multi(P0, f.t_r, T, out=pi, ws=ws); ts.append(time.perf_counter() - t0)
print("stationary_multi with out/ws given: %.1f us" % (np.median(ts) * 1e6))
ts = []
for _ in range(200):
    t0 = time.perf_counter(); torch.cuda.current_stream().synchronize(); ts.append(time.perf_counter() - t0)
print("bare sync: %.1f us" % (np.median(ts) * 1e6))
