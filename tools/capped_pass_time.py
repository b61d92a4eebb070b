"""Per-pass time of the c5 fp64 GEMV under sustained load (the board's power cap), by the number of
running vectors: a plan on c5's stored P~0 with V dead times and max_iter = 16 (nothing converges, so
every pass carries all V vectors), launched back to back for ~3 s; the GEMV time is the library's own
device stamps (splidar_plan_gemv_time). Run on the GPU box: python tools/capped_pass_time.py"""
import json
import subprocess
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2509_20500_b200 as spl  # noqa: E402
from workloads.configs import config  # noqa: E402


def smi():
    out = subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm,power.draw", "--format=csv,noheader,nounits"],
                         capture_output=True, text=True).stdout.strip().split(",")
    return float(out[0]), float(out[1])


w = config(5)
f = w.items[0].flux
P0 = spl.build_base(f, torch.float64)
tds = [it.t_d for it in w.items] + [it.t_d for it in w.sweep]
rows = []
for V in (17, 16, 9, 8, 4, 1):
    plan = spl.Plan(P0, f.t_r, [tds[:V]], tol=1e-12, max_iter=16)
    for _ in range(3):
        plan.launch()
    torch.cuda.synchronize()
    plan.gemv_time(reset=True)
    t0 = time.time()
    clk = []
    n = 0
    while time.time() - t0 < 3.0:
        for _ in range(8):
            plan.launch()
        n += 8
        torch.cuda.synchronize()
        clk.append(smi())
    sec, launches = plan.gemv_time()
    info = plan.info(check=False)
    rows.append({"V": V, "gemv": plan.gemv(), "us_per_pass": sec / launches * 1e6, "passes": launches,
                 "iters": int(info[0]["iters"]), "sm_mhz_median": float(np.median([c[0] for c in clk])),
                 "power_w_max": max(c[1] for c in clk),
                 "GBps": P0.numel() * 8 / (sec / launches) / 1e9})
    print(json.dumps(rows[-1]), flush=True)
    plan.close()
