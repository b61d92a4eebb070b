"""Row shards of one matrix on one GPU: the library's shard steps (partial GEMV over
a row block, the caller's all-reduce, replicated check) driven for W simulated ranks in one process,
the all-reduce done as a plain sum of the W partial products in rank order. Every rank must hold the
same pi, equal to the unsharded plan's to rounding (the sum order over rows differs), with the same
iteration counts +-1, and the oracle's Eq. 4 residual must vanish (pi P~ = pi).

(Running W ranks whose kernels wait on one another on one GPU is not possible; here every step of
every rank completes before the next starts, so nothing waits.)"""
import numpy as np
import pytest
import torch

import oracle
from workloads import config
from paper_2509_20500_b200.shard import row_block, sharded_solve

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def spl():
    assert torch.cuda.is_available(), "GPU tests need a B200"
    from paper_2509_20500_b200 import build
    build.build()
    import paper_2509_20500_b200 as s
    return s


def _sharded(spl, f, tds, W, dtype):
    N = f.n_bins
    plans = []
    for r in range(W):
        r0, n = row_block(N, r, W)
        rows = spl.build_base_rows(f, r0, n, dtype)
        plans.append(spl.ShardPlan(rows, r0, N, f.t_r, tds, tol=1e-12))
    for p in plans:
        p.init()
    it = 0
    while True:
        for p in plans:
            p.gemv()
        s = plans[0].ypart.clone()
        for p in plans[1:]:
            s += p.ypart                                   # the all-reduce, rank order
        for p in plans:
            p.ypart.copy_(s)
        more = [p.check() for p in plans]
        assert len(set(more)) == 1                         # replicated convergence decision
        it += 1
        if not more[0]:
            break
    infos = [p.finish() for p in plans]
    pis = [p.pi.detach().cpu().numpy().copy() for p in plans]
    for p in plans:
        p.close()
    return pis, infos


def test_build_base_rows_equals_full(spl):
    f = config(4).items[0].flux
    full = spl.build_base(f, torch.float64)
    for r0, n in ((0, 1000), (5000, 3001), (16384 - 7, 7)):
        rows = spl.build_base_rows(f, r0, n, torch.float64)
        assert torch.equal(rows, full[r0:r0 + n])


@pytest.mark.parametrize("W,N,V,dtype", [(2, 4096, 17, torch.float64), (3, 5000, 4, torch.float64),
                                         (4, 8192, 1, torch.float32), (8, 16384, 8, torch.float64)])
def test_sharded_equals_unsharded(spl, W, N, V, dtype):
    from workloads import Flux
    f0 = config(5).items[0].flux
    f = Flux(f0.t_r, N, f0.tau, f0.sigma, f0.signal, f0.background)
    w = config(5)
    tds = ([w.items[0].t_d] + [it.t_d for it in w.sweep])[:V]
    pis, infos = _sharded(spl, f, tds, W, dtype)
    for p in pis[1:]:
        assert np.array_equal(p, pis[0])
    P0 = spl.build_base(f, dtype)
    plan = spl.Plan(P0, f.t_r, np.array([tds]), tol=1e-12)
    ref_inf = plan.execute()
    ref = plan.pi[0].detach().cpu().numpy()
    plan.close()
    assert np.max(np.sum(np.abs(pis[0] - ref), axis=1)) <= 1e-13
    for a, b in zip(infos[0], ref_inf):
        assert a["converged"] and abs(a["iters"] - b["iters"]) <= 1 and a["shift_l"] == b["shift_l"]
    if N <= 5000:
        y = oracle.left_matvec_streamed(f, tds[0], pis[0][0])
        assert np.sum(np.abs(y - pis[0][0])) <= (1e-11 if dtype == torch.float64 else 1e-5)


def test_sharded_solve_helper_world1(spl):
    """shard.sharded_solve with a no-op all-reduce (world size 1) is the plain solve."""
    f = config(4).items[0].flux
    rows = spl.build_base_rows(f, 0, f.n_bins, torch.float64)
    plan = spl.ShardPlan(rows, 0, f.n_bins, f.t_r, [f.t_r * 1.2], tol=1e-12)
    infos = sharded_solve(plan, lambda t: None)
    P0 = spl.build_base(f, torch.float64)
    pi, info = spl.stationary(P0, f.t_r, f.t_r * 1.2)
    assert infos[0]["converged"] and np.sum(np.abs(plan.pi[0].cpu().numpy() - pi.cpu().numpy())) <= 1e-13
    plan.close()


def test_shard_rejects(spl):
    f = config(1).items[0].flux
    rows = spl.build_base_rows(f, 0, 10, torch.float64)
    with pytest.raises(spl.SplidarError):
        spl.build_base_rows(f, 250, 10, torch.float64)       # rows beyond N
    with pytest.raises(spl.SplidarError):
        spl.ShardPlan(rows, 250, f.n_bins, f.t_r, [75.0])    # row0 + n > N
