"""c5 plan: CUDA-graph WHILE loop vs eager host loop (same kernels), device time per solve (scratch)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2509_20500_b200 as spl
import bench
w, groups = bench.workload_items("c5")
f, tds = groups[0]
P0 = spl.build_base(f)
def timeit(plan, reps=3):
    plan.launch(); torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); plan.launch(); b.record(); torch.cuda.synchronize(); ts.append(a.elapsed_time(b))
    return min(ts), plan.info()
g = spl.Plan(P0, f.t_r, np.array([tds]))
tg, ig = timeit(g)
os.environ["SPLIDAR_EAGER"] = "1"
e = spl.Plan(P0, f.t_r, np.array([tds]))
te, ie = timeit(e)
it = max(i["iters"] for i in ig)
print(f"graph {tg:.2f} ms, eager {te:.2f} ms, iterations {it}, graph per iteration {tg/it*1e3:.1f} us")
# single GEMV pass time in a sustained loop: a plan with max_iter=1 repeated
os.environ.pop("SPLIDAR_EAGER")
one = spl.Plan(P0, f.t_r, np.array([tds]), max_iter=1)
one.launch(); torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(20): one.launch()
b.record(); torch.cuda.synchronize()
print(f"max_iter=1 plan (init + 1 GEMV + 1 check + finish): {a.elapsed_time(b)/20*1e3:.1f} us per launch")
