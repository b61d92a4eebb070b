"""Quick per-config run of the GPU path with bounded iterations and timings (development aid)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2509_20500_b200 as spl
from workloads import config

def t(fn):
    torch.cuda.synchronize(); a = time.perf_counter(); r = fn(); torch.cuda.synchronize(); return r, time.perf_counter() - a

for k in [int(x) for x in (sys.argv[1:] or "1 2 3 4 5".split())]:
    w = config(k)
    for dt in (torch.float64, torch.float32):
        for it in w.items[:2]:
            f = it.flux
            ws = spl.workspace(f.n_bins)
            P0, tb = t(lambda: spl.build_base(f, dt, ws=ws))
            P0, tb = t(lambda: spl.build_base(f, dt, out=P0, ws=ws))
            (pi, info), ts = t(lambda: spl.stationary(P0, f.t_r, it.t_d, max_iter=300, ws=ws, check=False))
            (pi, info), ts = t(lambda: spl.stationary(P0, f.t_r, it.t_d, max_iter=300, ws=ws, check=False))
            nb = f.n_bins ** 2 * P0.element_size()
            print(f"c{k} {str(dt)[6:]} N={f.n_bins} build {tb*1e3:.3f} ms ({nb/tb/1e9:.0f} GB/s)  solve {ts*1e3:.3f} ms "
                  f"iters={info['iters']} conv={info['converged']} ch={info['l1_change']:.2e} "
                  f"GEMV {info['iters']*nb/ts/1e9:.0f} GB/s", flush=True)
            del P0; torch.cuda.empty_cache()
