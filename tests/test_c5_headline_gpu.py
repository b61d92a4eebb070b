"""The headline configuration (c5, the bench's default step) checked against the oracle itself.

c5: N = 32768, t_r = 200, two returns, B = 0.8; the bench step solves t_d = 430 plus the 16-value
dead-time sweep on one P~0 (17 vectors in one multi-vector plan), in fp64 and in fp32 storage, and
the same 17 items on the structured operator (f2). Every pi is checked by the residual of the
ORACLE's own Eq. 4 matrix (dead time inside the integral bounds), streamed row by row:
||pi P~_eq4 - pi||_1 (pi P~ = pi). The oracle never stores the 8.6 GB matrix; it recomputes
each Eq. 4 row once per dead time and applies it to all solutions of that dead time.

Tolerances: fp64 1e-11 (the power iteration stops at an L1 change of 1e-12 with |lambda_2| < 1,
so the residual of the exact fixed point is ~1e-12 plus rounding); fp32 storage 1e-5 (the fp32
matrix's own fixed point, BASELINE.json fp32 tolerance).
"""
import numpy as np
import pytest
import torch

import oracle
from workloads import config

pytestmark = pytest.mark.gpu

TDS_CHECKED = (430.0, 10.0, 206.0, 500.0)   # the single solve + both sweep ends + a frac(u) = 0.04 case


@pytest.fixture(scope="module")
def spl():
    assert torch.cuda.is_available(), "GPU tests need a B200"
    from paper_2509_20500_b200 import build
    build.build()
    import paper_2509_20500_b200 as s
    return s


def _bench_plan_pis(spl, f, tds, dtype):
    """The bench's c5 step: one building plan (build P~0 + iteration 1 from its column sums + the
    power iteration), all dead times as one multi-vector plan; fp32 runs on the encoded storage and
    the int8 tensor-core GEMV, fp64 on the FP64 tensor cores."""
    P0 = spl.empty_matrix(f.n_bins, dtype, n_matrices=1)
    plan = spl.Plan(P0, f.t_r, np.array([tds]), tol=1e-12, build=[f])
    infos = plan.execute(check=dtype == torch.float64)
    if dtype == torch.float32:
        assert plan.gemv() == "tensor_i8" and plan.storage() == "encoded"
    else:
        assert plan.gemv() == "fp64" and plan.storage() == "ieee"
    pis = plan.pi[0].detach().cpu().numpy().copy()
    plan.close()
    del P0
    torch.cuda.empty_cache()
    return pis, infos


def test_config5_headline_vs_oracle_residual(spl):
    w = config(5)
    f = w.items[0].flux
    tds = [w.items[0].t_d] + [it.t_d for it in w.sweep]
    assert all(td in tds for td in TDS_CHECKED)
    pi64, inf64 = _bench_plan_pis(spl, f, tds, torch.float64)
    pi32, inf32 = _bench_plan_pis(spl, f, tds, torch.float32)
    shape, S, B = spl.flux_items(f)
    pis, infs = spl.stationary_structured(shape, np.repeat(S, len(tds)), np.repeat(B, len(tds)), tds)
    pis = pis.detach().cpu().numpy()
    for inf in (inf64, inf32, infs):
        assert all(i["converged"] for i in inf)
        assert [i["shift_l"] for i in inf] == [oracle.shift_l(f, td) for td in tds]
    for td in TDS_CHECKED:
        v = tds.index(td)
        X = np.stack([pi64[v], pis[v], pi32[v]])
        Y = oracle.left_matvec_streamed_multi(f, td, X)
        res = np.sum(np.abs(Y - X), axis=1)
        assert res[0] <= 1e-11, (td, "fp64 dense", res[0])
        assert res[1] <= 1e-11, (td, "structured", res[1])
        assert res[2] <= 1e-5, (td, "fp32 dense", res[2])
        # and the two fp64 routes agree with each other to the pi tolerance
        assert np.sum(np.abs(pi64[v] - pis[v])) <= 1e-10, td
