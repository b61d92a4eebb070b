"""GPU vs oracle over seeded random theta (pytest -m gpu): a sweep beyond the fixed parity cases,
drawn like the paper's workloads (narrow Gaussian returns on a flat floor, 0-2 pulses, S in [0, 10],
B in [1e-3, 5], sigma 0.3-5 bins, dead times anywhere in three periods plus exact whole bins and
whole periods), at sizes that cross the solver boundaries: N <= 2048 runs the fused cluster solver
(resident or L2-streamed rows), N > 2048 the graph path, ragged N everywhere. Per draw: P~0 entries
(max-abs) and row sums, the dead-time permutation against the oracle's direct Eq. 4 (raw t_d in
the bounds; Theorem 2), and pi by the plan (one vector per dead time, all dead
times of a draw in one multi-vector plan) against the oracle's stationary vector.
Tolerances: BASELINE.json north_star (fp64 entries 1e-12, rows 1e-12, pi 1e-10 L1; fp32 1e-5)."""
import numpy as np
import pytest
import torch

import oracle
from workloads import Flux

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def spl():
    assert torch.cuda.is_available(), "GPU tests need a B200"
    from paper_2509_20500_b200 import build
    build.build()
    import paper_2509_20500_b200 as s
    return s


def _draw(seed, n):
    rng = np.random.default_rng(seed)
    t_r = float(rng.choice([100.0, 200.0, 64.0]))
    k = int(rng.integers(0, 3))
    d = t_r / n
    f = Flux(t_r, n, tuple(float(x) for x in rng.uniform(0.0, t_r, k)),
             tuple(float(x) for x in rng.uniform(0.3 * d, 5.0 * d, k)),
             tuple(float(x) for x in rng.uniform(0.0, 10.0, k)), float(np.exp(rng.uniform(np.log(1e-3), np.log(5.0)))))
    m = int(rng.integers(0, 3 * n))
    tds = [float(rng.uniform(0.0, 3.0 * t_r)), m * d, float(m % 4) * t_r]
    return f, tds


def _oracle_pi(P):
    if P.shape[0] <= 1100:
        return oracle.stationary_dense(P)
    pi, _, _, ok = oracle.stationary_power(P, 1e-15)
    assert ok
    return pi


SIZES = [2, 5, 33, 97, 255, 256, 511, 1000, 1029, 2047, 2048, 2049, 2311, 3001]


@pytest.mark.parametrize("i,n", list(enumerate(SIZES)))
def test_random_theta_f64(spl, i, n):
    f, tds = _draw(9100 + i, n)
    P0 = spl.build_base(f, torch.float64)
    got = P0.cpu().numpy()
    assert np.max(np.abs(got - oracle.build_eq4(f, 0.0))) <= 1e-12
    assert np.max(np.abs(got.sum(axis=1) - 1.0)) <= 1e-12
    P = spl.apply_deadtime(P0, f.t_r, tds[0])
    Pe = oracle.build_eq4(f, tds[0])
    assert np.max(np.abs(P.cpu().numpy() - Pe)) <= 1e-12
    plan = spl.Plan(P0, f.t_r, np.array([tds]), tol=1e-12)
    infos = plan.execute(check=False)
    pis = plan.pi.cpu().numpy()[0]
    for v, td in enumerate(tds):
        assert infos[v]["converged"], (n, td, infos[v])
        assert infos[v]["shift_l"] == oracle.shift_l(f, td)
        want = _oracle_pi(Pe if v == 0 else oracle.build_eq4(f, td))
        assert np.sum(np.abs(pis[v] - want)) <= 1e-10, (n, td)
    plan.close()


@pytest.mark.parametrize("i,n", list(enumerate(SIZES[::2])))
def test_random_theta_f32(spl, i, n):
    f, tds = _draw(9300 + i, n)
    P0 = spl.build_base(f, torch.float32)
    got = P0.cpu().numpy().astype(np.float64)
    assert np.max(np.abs(got - oracle.build_eq4(f, 0.0))) <= 1e-5
    plan = spl.Plan(P0, f.t_r, np.array([tds]), tol=1e-12, max_iter=100000)
    plan.execute(check=False)
    pis = plan.pi.cpu().numpy()[0]
    for v, td in enumerate(tds):
        assert np.sum(np.abs(pis[v] - _oracle_pi(oracle.build_eq4(f, td)))) <= 1e-5, (n, td)
    plan.close()
