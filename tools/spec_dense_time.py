"""Time splidar_second_eigenvalue_dense at config 4 / 5 (N = 16384 / 32768, fp64 and fp32 storage):
products per solve, ms per solve (CUDA events, warm), and the GEMV stream rate N^2 * sizeof(T) per
product. Prints one JSON line per case. Usage: python tools/spec_dense_time.py"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2509_20500_b200 as spl  # noqa: E402
from workloads import config  # noqa: E402


def main():
    for k in (4, 5):
        it = config(k).items[0]
        f = it.flux
        for dt in (torch.float64, torch.float32):
            P0 = spl.build_base(f, dt)
            pi, _ = spl.stationary(P0, f.t_r, it.t_d)
            info = spl.second_eigenvalue_dense(P0, f.t_r, it.t_d, pi)   # warm (graph build, attributes)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            reps = 3
            torch.cuda.synchronize()
            e0.record()
            for _ in range(reps):
                info = spl.second_eigenvalue_dense(P0, f.t_r, it.t_d, pi)
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / reps
            n = f.n_bins
            per = ms / info["iters"]
            print(json.dumps({"config": k, "N": n, "dtype": str(dt).split(".")[-1], "iters": info["iters"],
                              "ms_per_solve": round(ms, 3), "us_per_product": round(per * 1e3, 2),
                              "stream_GBps": round(n * n * P0.element_size() / (per * 1e-3) / 1e9, 1),
                              "modulus": info["modulus"], "phase": info["phase"]}))


if __name__ == "__main__":
    main()
