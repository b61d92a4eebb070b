"""Sustained (not serialised, not cache-flushed) per-kernel device times of the c5 solve, from CUPTI
activity records via torch.profiler: compares the GEMV inside the WHILE loop with its isolated ncu
time (scratch; numbers go to DESIGN.md)."""
import os
import sys
import collections

import numpy as np
import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2509_20500_b200 as spl  # noqa: E402
import bench  # noqa: E402

w, groups = bench.workload_items("c5")
f, tds = groups[0]
P0 = spl.build_base(f)
plan = spl.Plan(P0, f.t_r, np.array([tds]))
plan.launch()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    e0.record()
    plan.launch()
    e1.record()
    torch.cuda.synchronize()
total = e0.elapsed_time(e1)
agg = collections.defaultdict(lambda: [0, 0.0, []])
evs = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
for e in evs:
    a = agg[e.name.split("(")[0][-40:]]
    a[0] += 1
    a[1] += e.device_time_total if hasattr(e, "device_time_total") else e.cuda_time_total
    a[2].append(e.time_range.start)
print(f"solve (events) {total:.3f} ms; iterations {max(i['iters'] for i in plan.info())}")
for k, (n, t, _) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{k:40s} {n:4d} {t / n:10.1f} us avg {t / 1e3:9.3f} ms")
starts = sorted((e.time_range.start, e.time_range.end, e.name[:30]) for e in evs)
gaps = [b[0] - a[1] for a, b in zip(starts, starts[1:])]
print(f"kernels {len(starts)}, busy {sum(e - s for s, e, _ in starts) / 1e3:.3f} ms, gaps sum {sum(gaps) / 1e3:.3f} ms, "
      f"median gap {np.median(gaps):.2f} us")
gemv = [e - s for s, e, n in starts if "power_step" in n]
print("GEMV per launch (us): first 5", [round(x, 1) for x in gemv[:5]], "last 5", [round(x, 1) for x in gemv[-5:]])
