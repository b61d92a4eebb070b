import os, sys, numpy as np, torch
sys.path.insert(0, '/root/repo')
import paper_2509_20500_b200 as spl
from workloads import config, Flux
for k, dt, V in ((5, torch.float64, 17), (5, torch.float32, 17), (4, torch.float64, 1), (3, torch.float64, 1), (1, torch.float64, 1), (2, torch.float64, 1)):
    w = config(k)
    if k in (1, 2, 3):
        fl = [it.flux for it in w.items]; T = np.array([[it.t_d] for it in w.items])
    else:
        fl = [w.items[0].flux]; T = np.array([([w.items[0].t_d] + [it.t_d for it in w.sweep])[:V]])
    N = fl[0].n_bins
    P0 = spl.empty_matrix(N, dt, n_matrices=len(fl))
    pa = spl.Plan(P0, fl[0].t_r, T, tol=1e-12, build=fl)
    ia = pa.execute(); pia = pa.pi.cpu().numpy()
    spl.build_base_batched(fl, dt, out=P0)
    pb = spl.Plan(P0, fl[0].t_r, T, tol=1e-12)
    ib = pb.execute(); pib = pb.pi.cpu().numpy()
    err = np.max(np.sum(np.abs(pia - pib), axis=-1))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for p in (pa,):
        for _ in range(3):
            e0.record(); p.launch(); e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
    tb = []
    for _ in range(3):
        e0.record(); spl.build_base_batched(fl, dt, out=P0); pb.launch(); e1.record(); torch.cuda.synchronize(); tb.append(e0.elapsed_time(e1))
    print(f"c{k} {dt} V={T.shape[1]} M={len(fl)} err {err:.2e} iters build-plan {[i['iters'] for i in ia][:5]} plain {[i['iters'] for i in ib][:5]} gemv {pa.gemv()} ms build-plan {min(ts):.3f} separate {min(tb):.3f}")
