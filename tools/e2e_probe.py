"""Host-side cost of each public call in bench.py's e2e step (building plans): mean wall time per call
over many steps. Diagnostic only (run via gpurun): python tools/e2e_probe.py c1"""
import sys, time
import torch
sys.path.insert(0, ".")
import bench

wl = sys.argv[1] if len(sys.argv) > 1 else "c1"
w, groups = bench.workload_items(wl, 0, 1)
st = bench.OurStep(groups, "f64", "factored")
N = st.N
pi_host = torch.empty((st.n_solves, N), dtype=torch.float64, pin_memory=True)
p = st.plans[0]
fl = st.fluxes
n = p.M * p.V
T = {k: 0.0 for k in ("set_fluxes", "launch", "copy", "info", "total")}
K = 2000
for it in range(K + 200):
    t0 = time.perf_counter()
    p.set_fluxes(fl)
    t1 = time.perf_counter()
    p.launch()
    t2 = time.perf_counter()
    pi_host[0:n].copy_(p.pi.reshape(n, N), non_blocking=True)
    t3 = time.perf_counter()
    p.info()
    t4 = time.perf_counter()
    if it >= 200:
        for k, v in zip(("set_fluxes", "launch", "copy", "info", "total"), (t1 - t0, t2 - t1, t3 - t2, t4 - t3, t4 - t0)):
            T[k] += v
print(wl, {k: round(v / K * 1e6, 2) for k, v in T.items()}, "us per step")
# launches only (no sync): host enqueue rate
torch.cuda.synchronize()
t0 = time.perf_counter()
for it in range(K):
    p.launch()
torch.cuda.synchronize()
print("launch-only loop", round((time.perf_counter() - t0) / K * 1e6, 2), "us per launch (device-bound if ~ device step)")
