"""The persistent loop kernel (k_power_loop: every power iteration of a plan in one cooperative launch,
GEMV pass + grid barrier + convergence check + grid barrier; P:79 iterated on the device) against the
two-kernel conditional-WHILE graph of the same plan (the default; the loop is opt-in with
SPLIDAR_PERSIST=1, see DESIGN.md §6 for the A/B that kept it opt-in): the same arithmetic in the
same order, so pi must be bit-identical and the infos (iterations, L1 change, convergence) equal, on
every solver shape the loop kernel takes (fp64 single vector on DFMA, DMMA groups with converging
vectors compacted, fp32 storage on DFMA, several matrices whose vectors stop at different passes,
building plans whose iteration 1 is the build's column sums, a ragged N and an ENOCONV stop).
The loop plans are also checked against the oracle's stationary vector (pytest -m gpu)."""
import numpy as np
import pytest
import torch

import oracle
from workloads import random_flux

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def spl():
    assert torch.cuda.is_available(), "GPU tests need a B200"
    from paper_2509_20500_b200 import build
    build.build()
    import paper_2509_20500_b200 as s
    return s


def _pair(spl, monkeypatch, make):
    """(loop plan, WHILE plan) built by make(); both executed."""
    monkeypatch.setenv("SPLIDAR_PERSIST", "1")
    a = make()
    monkeypatch.delenv("SPLIDAR_PERSIST")
    b = make()
    ia = a.execute(check=False)
    ib = b.execute(check=False)
    return a, b, ia, ib


@pytest.mark.parametrize("dtype,N,nv", [(torch.float64, 3000, 1), (torch.float64, 3000, 5),
                                        (torch.float64, 4096, 17), (torch.float64, 9001, 8),
                                        (torch.float32, 3000, 1), (torch.float64, 3000, 32)])
def test_loop_equals_while_graph(spl, monkeypatch, dtype, N, nv):
    f = random_flux(np.random.default_rng(7000 + N + nv), N, 2)
    tds = [float(x) for x in np.linspace(3.0, 290.0, nv)]
    P0 = spl.build_base(f, dtype)
    a, b, ia, ib = _pair(spl, monkeypatch, lambda: spl.Plan(P0, f.t_r, np.array([tds]), tol=1e-12))
    assert a.kind == "loop" and b.kind == "graph"
    assert torch.equal(a.pi, b.pi)
    assert ia == ib and all(i["converged"] for i in ia)
    a.close()
    b.close()


def test_loop_several_matrices_and_oracle(spl, monkeypatch):
    """Four matrices x 3 dead times: matrices leave the active list at different passes; pi against the
    oracle's stationary vector of P~ = J_l P~0 built from its own Eq. 4 (dead time in the bounds)."""
    rng = np.random.default_rng(99)
    N = 2304
    fl = [random_flux(rng, N, k) for k in (1, 2, 1, 2)]
    T = np.array([[5.0, 40.0, 95.0], [130.0, 7.5, 60.0], [20.0, 20.5, 250.0], [0.0, 80.0, 160.0]])
    P0 = spl.build_base_batched(fl, torch.float64)
    a, b, ia, ib = _pair(spl, monkeypatch, lambda: spl.Plan(P0, fl[0].t_r, T, tol=1e-12))
    assert a.kind == "loop"
    assert torch.equal(a.pi, b.pi) and ia == ib
    iters = [i["iters"] for i in ia]
    assert len(set(iters)) > 1
    pi = a.pi.cpu().numpy()
    for m in (0, 3):
        for v in (0, 2):
            P = oracle.build_eq4(fl[m], float(T[m, v]))
            ref = oracle.stationary_dense(P) if N <= 1100 else oracle.stationary_power(P, 1e-15)[0]
            assert np.sum(np.abs(pi[m, v] - ref)) <= 1e-10, (m, v)
    a.close()
    b.close()


@pytest.mark.parametrize("dtype", [torch.float64, torch.float32])
def test_loop_building_plan(spl, monkeypatch, dtype):
    """Building plans: steps 1-2 and iteration 1 (column sums) before the loop kernel; fp32 with 3 dead
    times stays off the int8 GEMV (it needs 8-18), so it runs the loop kernel too."""
    rng = np.random.default_rng(5)
    N = 4096
    fl = [random_flux(rng, N, 2), random_flux(rng, N, 1)]
    T = np.array([[10.0, 44.0, 130.0], [3.0, 60.0, 99.0]])
    P = spl.empty_matrix(N, dtype, n_matrices=2)
    Q = spl.empty_matrix(N, dtype, n_matrices=2)
    monkeypatch.setenv("SPLIDAR_PERSIST", "1")
    a = spl.Plan(P, fl[0].t_r, T, tol=1e-12, build=fl)
    monkeypatch.delenv("SPLIDAR_PERSIST")
    b = spl.Plan(Q, fl[0].t_r, T, tol=1e-12, build=fl)
    assert a.kind == "loop" and b.kind == "graph"
    for _ in range(2):   # relaunch: the loop kernel's barrier and counters reset per launch
        ia = a.execute(check=False)
        ib = b.execute(check=False)
        assert torch.equal(a.pi, b.pi) and ia == ib
        assert torch.equal(P, Q)
    a.close()
    b.close()


def test_loop_max_iter_stop(spl, monkeypatch):
    """max_iter reached inside the loop kernel: ENOCONV state, same last iterate as the WHILE graph."""
    f = random_flux(np.random.default_rng(11), 3000, 2)
    P0 = spl.build_base(f, torch.float64)
    mk = lambda: spl.Plan(P0, f.t_r, np.array([[17.0, 170.0]]), tol=1e-30, max_iter=7)
    a, b, ia, ib = _pair(spl, monkeypatch, mk)
    assert torch.equal(a.pi, b.pi) and ia == ib
    assert all(i["iters"] == 7 and not i["converged"] for i in ia)
    a.close()
    b.close()
