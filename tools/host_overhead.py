"""Host-side cost of the public structured API on the 8192-item grid (scratch measurement)."""
import sys, os, time, ctypes as C
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2509_20500_b200 as spl
from paper_2509_20500_b200 import splidar as S_
import bench
w, groups = bench.workload_items("grid")
sg = bench._shape_groups(groups)
shape, S, B, T = sg[0]
S, B, T = np.array(S), np.array(B), np.array(T)
for _ in range(3):
    pi, inf = spl.stationary_structured(shape, S, B, T)
torch.cuda.synchronize()
t0 = time.perf_counter(); pi, inf = spl.stationary_structured(shape, S, B, T); torch.cuda.synchronize(); t1 = time.perf_counter()
print("full call ms", (t1 - t0) * 1e3)
t0 = time.perf_counter(); x = S_._items(shape, S, B, T); t1 = time.perf_counter(); print("_items ms", (t1 - t0) * 1e3)
t0 = time.perf_counter(); ws = spl.structured_workspace(256, 4096, 8192); torch.cuda.synchronize(); t1 = time.perf_counter(); print("workspace ms", (t1 - t0) * 1e3)
M = S.size
pi = torch.empty((M, 256), dtype=torch.float64, device="cuda")
infos = (S_.SolveInfo * M)()
fa = S_._FluxArg(shape)
t0 = time.perf_counter()
st = S_._lib().splidar_stationary_structured(C.byref(fa.s), M, S.ctypes.data, B.ctypes.data, T.ctypes.data, 1e-12, 10**6,
                                             pi.data_ptr(), ws.data_ptr(), ws.numel(), infos, S_._stream(None))
t1 = time.perf_counter(); print("C call (incl. kernel + sync) ms", (t1 - t0) * 1e3, st)
t0 = time.perf_counter(); d = [i.as_dict() for i in infos]; t1 = time.perf_counter(); print("as_dict ms", (t1 - t0) * 1e3)
pl = spl.StructPlan("solve", shape, S, B, T)
pl.launch(); pl.info()
t0 = time.perf_counter(); pl.launch(); torch.cuda.synchronize(); t1 = time.perf_counter(); print("plan launch+sync ms", (t1 - t0) * 1e3)
t0 = time.perf_counter(); r = pl.info(); t1 = time.perf_counter(); print("plan info ms", (t1 - t0) * 1e3, r[1])
t0 = time.perf_counter(); pl2 = spl.StructPlan("solve", shape, S, B, T); torch.cuda.synchronize(); t1 = time.perf_counter(); print("plan create ms", (t1 - t0) * 1e3)
