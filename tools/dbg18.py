import os, sys, numpy as np, torch
sys.path.insert(0, '/root/repo')
import paper_2509_20500_b200 as spl
from workloads import Flux, config
os.environ["SPLIDAR_FUSED"]="0"
N=int(sys.argv[1]); V=int(sys.argv[2])
w=config(5); f0=w.items[0].flux
f=Flux(f0.t_r,N,f0.tau,f0.sigma,f0.signal,f0.background)
tds=([w.items[0].t_d]+[it.t_d for it in w.sweep]+[333.3, 20.0, 55.5])[:V]
P0=spl.build_base(f, torch.float32)
for env in ("1","0"):
    os.environ["SPLIDAR_I8"]=env
    plan=spl.Plan(P0,f.t_r,np.array([tds]),tol=1e-12,max_iter=200)
    inf=plan.execute(check=False)
    print(env, plan.gemv(), [i["iters"] for i in inf], ["%.1e"%i["l1_change"] for i in inf][-3:])
    pi=plan.pi.cpu().numpy(); print("  sum", pi.sum(axis=-1)[0][-3:], "min", pi.min())
    plan.close()
