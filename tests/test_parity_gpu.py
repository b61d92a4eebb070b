"""GPU path vs the CPU oracle, element by element, through the C ABI (pytest -m gpu).

Tolerances (BASELINE.json north_star): fp64 entries <= 1e-12 max-abs, row sums within 1e-12 of 1,
pi <= 1e-10 in L1; fp32 storage <= 1e-5 (entries and pi). The oracle builds P~ entry by entry from
Eq. 4 with the dead time inside the integral bounds; the GPU builds the base matrix from
the paper's reparameterised form (§3.4) and applies the dead time as the row permutation of
Theorem 2, so every comparison below also checks Theorem 2 (exact after normalisation, R1).
"""
import math

import numpy as np
import pytest
import torch

import oracle
from workloads import Flux, config, parity_cases, random_flux

from ._structured import oracle_vectors, sampled_rows, structured_pi

pytestmark = pytest.mark.gpu

TOL_E64, TOL_ROW, TOL_PI64 = 1e-12, 1e-12, 1e-10
TOL_E32, TOL_PI32 = 1e-5, 1e-5


@pytest.fixture(scope="module")
def spl():
    assert torch.cuda.is_available(), "GPU tests need a B200"
    from paper_2509_20500_b200 import build
    build.build()
    import paper_2509_20500_b200 as s
    return s


def _np(t):
    return t.detach().cpu().numpy()


def _oracle_pi(P):
    n = P.shape[0]
    if n <= 1100:
        return oracle.stationary_dense(P)
    pi, _, _, ok = oracle.stationary_power(P, 1e-15)
    assert ok
    return pi


CASES = parity_cases()
IDS = [f"N{c.flux.n_bins}-K{c.flux.n_pulses}-td{c.t_d:.2f}" for c in CASES]


# ------------------------------------------------------------- a1-a2: flux vectors and the scan
@pytest.mark.parametrize("case", CASES + [config(k).items[0] for k in range(1, 6)],
                         ids=IDS + [f"config{k}" for k in range(1, 6)])
def test_flux_vectors(spl, case):
    f = case.flux
    v = spl.flux_vectors(f)
    lam, F, Lam = oracle_vectors(f)
    tolF = 1e-13 * max(1.0, Lam)
    assert abs(_np(v["Lambda"])[0] - Lam) <= tolF
    assert np.max(np.abs(_np(v["F"]) - F)) <= tolF
    assert np.max(np.abs(_np(v["lam"]) - lam) / lam) <= 1e-13


# ------------------------------------------------------------- a3-a4: base matrix
@pytest.mark.parametrize("mode", ["factored", "exp"])
@pytest.mark.parametrize("case", CASES, ids=IDS)
def test_build_base_f64(spl, case, mode):
    f = case.flux
    P0 = spl.build_base(f, torch.float64, mode)
    got = _np(P0)
    want = oracle.build_eq4(f, 0.0)
    assert np.max(np.abs(got - want)) <= TOL_E64
    assert np.max(np.abs(got.sum(axis=1) - 1.0)) <= TOL_ROW


@pytest.mark.parametrize("mode", ["factored", "exp"])
@pytest.mark.parametrize("case", CASES[::3], ids=IDS[::3])
def test_build_base_f32(spl, case, mode):
    f = case.flux
    got = _np(spl.build_base(f, torch.float32, mode)).astype(np.float64)
    want = oracle.build_eq4(f, 0.0)
    assert np.max(np.abs(got - want)) <= TOL_E32
    assert np.max(np.abs(got.sum(axis=1) - 1.0)) <= 1e-4


# ------------------------------------------------------------- a5: dead time as row permutation
@pytest.mark.parametrize("case", CASES, ids=IDS)
def test_apply_deadtime_equals_eq4(spl, case):
    """J_l P~0 on the GPU == the oracle's direct Eq. 4 with t_d inside the bounds."""
    f = case.flux
    P0 = spl.build_base(f, torch.float64)
    P = spl.apply_deadtime(P0, f.t_r, case.t_d)
    assert np.max(np.abs(_np(P) - oracle.build_eq4(f, case.t_d))) <= TOL_E64


def test_apply_deadtime_f32_exact_copy(spl):
    f = CASES[10].flux
    P0 = spl.build_base(f, torch.float32)
    P = spl.apply_deadtime(P0, f.t_r, 37.0)
    l = spl.shift(f.t_r, f.n_bins, 37.0)
    assert torch.equal(P, torch.roll(P0, -l, dims=0))


# ------------------------------------------------------------- a6: power iteration
@pytest.mark.parametrize("case", CASES, ids=IDS)
def test_stationary_f64(spl, case):
    f = case.flux
    P0 = spl.build_base(f, torch.float64)
    pi, info = spl.stationary(P0, f.t_r, case.t_d, tol=1e-12)
    assert info["converged"] and info["l1_change"] < 1e-12
    assert info["shift_l"] == oracle.shift_l(f, case.t_d)
    want = _oracle_pi(oracle.build_eq4(f, case.t_d))
    got = _np(pi)
    assert np.sum(np.abs(got - want)) <= TOL_PI64
    assert abs(got.sum() - 1.0) <= 1e-13 and np.all(got > 0)


@pytest.mark.parametrize("case", CASES[1::3], ids=IDS[1::3])
def test_stationary_f32(spl, case):
    f = case.flux
    P0 = spl.build_base(f, torch.float32)
    pi, info = spl.stationary(P0, f.t_r, case.t_d, tol=1e-12, max_iter=100000, check=False)
    want = _oracle_pi(oracle.build_eq4(f, case.t_d))
    assert np.sum(np.abs(_np(pi) - want)) <= TOL_PI32


def test_stationary_noconv_reported(spl):
    f = config(1).items[0].flux
    P0 = spl.build_base(f)
    with pytest.raises(spl.SplidarError) as e:
        spl.stationary(P0, f.t_r, 75.0, tol=1e-12, max_iter=2)
    assert e.value.status == spl.ENOCONV
    pi, info = spl.stationary(P0, f.t_r, 75.0, tol=1e-12, max_iter=2, check=False)
    assert info["iters"] == 2 and not info["converged"] and info["l1_change"] > 1e-12
    # pi holds the second iterate: compare with two oracle power steps
    P = oracle.build_eq4(f, 75.0)
    x = np.full(f.n_bins, 1.0 / f.n_bins)
    for _ in range(2):
        x = x @ P
        x /= x.sum()
    assert np.sum(np.abs(_np(pi) - x)) <= 1e-13


def test_deterministic(spl):
    f = config(2).items[5].flux
    P0a = spl.build_base(f)
    P0b = spl.build_base(f)
    assert torch.equal(P0a, P0b)
    pa, _ = spl.stationary(P0a, f.t_r, 50.0)
    pb, _ = spl.stationary(P0b, f.t_r, 50.0)
    assert torch.equal(pa, pb)


def test_plan_reuse_and_multivector(spl):
    """One P~0, several dead times in one multi-vector plan, executed twice: identical results,
    each vector equal to its single-vector solve and to the oracle."""
    f = random_flux(np.random.default_rng(3), 777, 2)
    tds = [0.0, 13.0, 55.5, 130.0, 299.0]
    P0 = spl.build_base(f)
    plan = spl.Plan(P0, f.t_r, np.array([tds]), tol=1e-12)
    i1 = plan.execute()
    p1 = plan.pi.clone()
    i2 = plan.execute()
    assert torch.equal(p1, plan.pi) and i1 == i2
    for v, td in enumerate(tds):
        single, info = spl.stationary(P0, f.t_r, td)
        assert info["iters"] == i1[v]["iters"]
        assert np.sum(np.abs(_np(plan.pi[0, v]) - _np(single))) <= 1e-14
        want = oracle.stationary_dense(oracle.build_eq4(f, td))
        assert np.sum(np.abs(_np(plan.pi[0, v]) - want)) <= TOL_PI64
    plan.close()


# ------------------------------------------------------------- BASELINE configs 1-3 (full)
def test_config1_full(spl):
    it = config(1).items[0]
    f = it.flux
    P0 = spl.build_base(f)
    P = spl.apply_deadtime(P0, f.t_r, it.t_d)
    want = oracle.build_eq4(f, it.t_d)
    assert np.max(np.abs(_np(P) - want)) <= TOL_E64
    pi, info = spl.stationary(P0, f.t_r, it.t_d)
    assert np.sum(np.abs(_np(pi) - oracle.stationary_dense(want))) <= TOL_PI64
    assert info["shift_l"] == 192


def test_config2_sweep(spl):
    w = config(2)
    # per-item pulse centres differ, so each item is its own shape: solve them through the batched
    # builder + one plan over 6 matrices
    fl = [it.flux for it in w.items]
    P0 = spl.build_base_batched(fl)
    plan = spl.Plan(P0, 100.0, np.array([[it.t_d] for it in w.items]), tol=1e-12)
    infos = plan.execute()
    for m, it in enumerate(w.items):
        want_P = oracle.build_eq4(it.flux, 0.0)
        assert np.max(np.abs(_np(P0[m]) - want_P)) <= TOL_E64
        want = oracle.stationary_dense(oracle.build_eq4(it.flux, it.t_d))
        assert np.sum(np.abs(_np(plan.pi[m, 0]) - want)) <= TOL_PI64
        assert infos[m]["converged"]
    plan.close()


def test_config3_sweep(spl):
    """64 (S, B) items at N = 4096 through splidar_sweep: all 64 vs the structured cross-check,
    4 of them element-wise against the oracle's Eq. 4 matrix and power iteration."""
    w = config(3)
    base = w.items[0].flux
    shape = Flux(base.t_r, base.n_bins, base.tau, base.sigma, (1.0,), 1.0)
    S = np.array([it.flux.signal[0] for it in w.items])
    B = np.array([it.flux.background for it in w.items])
    T = np.array([it.t_d for it in w.items])
    pi, infos = spl.sweep(shape, S, B, T, n_store=64)
    got = _np(pi)
    for m, it in enumerate(w.items):
        assert infos[m]["converged"]
        ref, _ = structured_pi(it.flux, it.t_d)
        assert np.sum(np.abs(got[m] - ref)) <= TOL_PI64, m
    for m in (0, 17, 42, 63):
        it = w.items[m]
        P = oracle.build_eq4(it.flux, it.t_d)
        want, _, _, ok = oracle.stationary_power(P, 1e-15)
        assert np.sum(np.abs(got[m] - want)) <= TOL_PI64


# ------------------------------------------------------------- configs 4-5 at full size
def _full_size_check(spl, flux, t_d, dtype, mode, tol_e, tol_pi, rows=None):
    N = flux.n_bins
    P0 = spl.build_base(flux, dtype, mode)
    torch.cuda.synchronize()
    l = oracle.shift_l(flux, t_d)
    rng = np.random.default_rng(N)
    rows = rows if rows is not None else sorted({0, 1, N - 1, l, (l + 1) % N, (N - l) % N, *rng.integers(0, N, 10)})
    # sampled rows of P~ = J_l P~0 against the oracle's Eq. 4 rows
    want = sampled_rows(flux, t_d, rows)
    got = np.stack([_np(P0[(r + l) % N]).astype(np.float64) for r in rows])
    assert np.max(np.abs(got - want)) <= tol_e
    # all row sums of P~0 on the device
    rs = _np(P0.sum(dim=1, dtype=torch.float64))
    assert np.max(np.abs(rs - 1.0)) <= (TOL_ROW if dtype == torch.float64 else 1e-4)
    pi, info = spl.stationary(P0, flux.t_r, t_d, tol=1e-12, check=dtype == torch.float64)
    got_pi = _np(pi)
    ref, _ = structured_pi(flux, t_d)
    assert np.sum(np.abs(got_pi - ref)) <= tol_pi
    del P0
    torch.cuda.empty_cache()
    return got_pi, info


def test_config4_full(spl):
    it = config(4).items[0]
    pi, info = _full_size_check(spl, it.flux, it.t_d, torch.float64, "factored", TOL_E64, TOL_PI64)
    assert info["converged"] and info["shift_l"] == 3277
    # residual against the oracle's own rows, streamed (pi P~ = pi)
    y = oracle.left_matvec_streamed(it.flux, it.t_d, pi)
    assert np.sum(np.abs(y - pi)) <= 1e-11


def test_config4_exp_mode(spl):
    it = config(4).items[0]
    _full_size_check(spl, it.flux, it.t_d, torch.float64, "exp", TOL_E64, TOL_PI64)


def test_config5_full_f64(spl):
    it = config(5).items[0]
    pi, info = _full_size_check(spl, it.flux, it.t_d, torch.float64, "factored", TOL_E64, TOL_PI64)
    assert info["converged"] and info["shift_l"] == 4916


@pytest.mark.parametrize("mode", ["factored", "exp"])
def test_config5_full_f32(spl, mode):
    it = config(5).items[0]
    _full_size_check(spl, it.flux, it.t_d, torch.float32, mode, TOL_E32, TOL_PI32)


@pytest.mark.parametrize("dtype,extra", [(torch.float64, False), (torch.float32, False), (torch.float64, True),
                                         (torch.float32, True)])
def test_config5_deadtime_sweep(spl, dtype, extra):
    """16 dead times on one P~0 in one multi-vector plan (the a7 sweep), each vs the structured pi;
    extra=True adds the t_d = 430 solve as a 17th vector (24-vector DMMA path, the bench's step)."""
    w = config(5)
    f = w.items[0].flux
    tds = [it.t_d for it in w.sweep] + ([w.items[0].t_d] if extra else [])
    P0 = spl.build_base(f, dtype)
    plan = spl.Plan(P0, f.t_r, np.array([tds]), tol=1e-12)
    infos = plan.execute(check=dtype == torch.float64)
    vec = oracle_vectors(f)
    tol = TOL_PI64 if dtype == torch.float64 else TOL_PI32
    for v, td in enumerate(tds):
        ref, _ = structured_pi(f, td, vectors=vec)
        assert np.sum(np.abs(_np(plan.pi[0, v]) - ref)) <= tol, td
        assert infos[v]["shift_l"] == oracle.shift_l(f, td)
    plan.close()
    del P0
    torch.cuda.empty_cache()


# ------------------------------------------------------------- degenerate cases
def test_constant_flux_uniform_pi(spl):
    """S = 0: circulant chain, pi = 1/N exactly, converges after one product (P5)."""
    f = Flux(100.0, 1000, (50.0,), (1.0,), (0.0,), 3.0)
    P0 = spl.build_base(f)
    pi, info = spl.stationary(P0, f.t_r, 75.0)
    assert np.max(np.abs(_np(pi) - 1e-3)) <= 1e-15
    assert info["iters"] <= 2


def test_tiny_n(spl):
    for n in (2, 3):
        f = random_flux(np.random.default_rng(n), n, 1)
        for td in (0.0, 10.0, 150.0):
            P0 = spl.build_base(f)
            pi, _ = spl.stationary(P0, f.t_r, td, tol=1e-14)
            want = oracle.stationary_dense(oracle.build_eq4(f, td))
            assert np.sum(np.abs(_np(pi) - want)) <= 1e-12


@pytest.mark.parametrize("nv", [3, 8, 9, 12, 17, 18, 24, 30, 32])
def test_multivector_counts(spl, nv):
    """Every compiled vector count (1..32 padded to 4/8/16/24/32), ragged N, each vector equal to its
    single-vector solve and to the oracle."""
    rng = np.random.default_rng(100 + nv)
    f = random_flux(rng, 601, 2)
    tds = [float(x) for x in rng.uniform(0, 3 * f.t_r, nv)]
    P0 = spl.build_base(f)
    plan = spl.Plan(P0, f.t_r, np.array([tds]), tol=1e-13)
    infos = plan.execute()
    for v in range(nv):
        assert infos[v]["converged"]
        single, info = spl.stationary(P0, f.t_r, tds[v], tol=1e-13)
        assert info["iters"] == infos[v]["iters"]
        assert np.sum(np.abs(_np(plan.pi[0, v]) - _np(single))) <= 1e-13
    for v in (0, nv - 1):
        want = oracle.stationary_dense(oracle.build_eq4(f, tds[v]))
        assert np.sum(np.abs(_np(plan.pi[0, v]) - want)) <= TOL_PI64
    plan.close()


# ------------------------------------------------------------- small-N fused solver vs the general path
@pytest.mark.parametrize("case", CASES[::2] + [config(1).items[0], config(2).items[3]],
                         ids=IDS[::2] + ["config1", "config2-item3"])
def test_fused_equals_general_path(spl, case, monkeypatch):
    """N <= 2048 plans run the fused cluster solver; the same plan forced onto the general graph path
    (SPLIDAR_FUSED=0) gives the same pi (<= 1e-14 L1) and iteration count (+-1), for fp64 and fp32."""
    f = case.flux
    for dt in (torch.float64, torch.float32):
        P0 = spl.build_base(f, dt)
        tds = [case.t_d, case.t_d + 7.3]
        fused = spl.Plan(P0, f.t_r, np.array([tds]), tol=1e-12)
        i_f = fused.execute(check=False)
        monkeypatch.setenv("SPLIDAR_FUSED", "0")
        general = spl.Plan(P0, f.t_r, np.array([tds]), tol=1e-12)
        monkeypatch.delenv("SPLIDAR_FUSED")
        i_g = general.execute(check=False)
        for v in range(2):
            assert abs(i_f[v]["iters"] - i_g[v]["iters"]) <= 1
            assert np.sum(np.abs(_np(fused.pi[0, v]) - _np(general.pi[0, v]))) <= 1e-13
        fused.close()
        general.close()


@pytest.mark.parametrize("n", [2, 37, 256, 700, 1024, 1537, 2048])
def test_fused_p2p_exchange_equals_cluster_barrier(spl, n, monkeypatch):
    """The fused solver's exchanges by st.async + per-CTA mbarriers (default) against the same solver
    with barrier.cluster exchanges (SPLIDAR_FUSED_P2P=0): the same sums in the same order, so pi is
    bit-identical and the infos equal; resident (N <= 384) and L2-streamed rows, several dead times."""
    f = random_flux(np.random.default_rng(4400 + n), n, 2)
    P0 = spl.build_base(f, torch.float64)
    T = np.array([[3.0, 61.5, 140.0]])
    monkeypatch.setenv("SPLIDAR_FUSED_1X", "0")          # both in the two-exchange form
    a = spl.Plan(P0, f.t_r, T, tol=1e-12)
    monkeypatch.setenv("SPLIDAR_FUSED_P2P", "0")
    b = spl.Plan(P0, f.t_r, T, tol=1e-12)
    monkeypatch.delenv("SPLIDAR_FUSED_P2P")
    monkeypatch.setenv("SPLIDAR_FUSED_LDG", "0")         # L2-streamed rows through the TMA ring
    c = spl.Plan(P0, f.t_r, T, tol=1e-12)
    monkeypatch.delenv("SPLIDAR_FUSED_LDG")
    monkeypatch.delenv("SPLIDAR_FUSED_1X")
    assert a.fused and b.fused and c.fused
    ia, ib, ic = a.execute(check=False), b.execute(check=False), c.execute(check=False)
    assert torch.equal(a.pi, b.pi) and ia == ib
    assert torch.equal(a.pi, c.pi) and ia == ic           # register loads == ring: same FMA order
    a.execute(check=False)                       # relaunch: the mbarrier phases start again
    assert torch.equal(a.pi, b.pi)
    for x in (a, b, c):
        x.close()


@pytest.mark.parametrize("n", [2, 37, 256, 700, 1024, 1537, 2048])
def test_fused_one_exchange_equals_two(spl, n, monkeypatch):
    """The default fused solver (one exchange per product: partials pushed straight to the CTA whose
    row they feed, s from the CTAs' partial totals) against the two-exchange form (owners sum and
    redistribute y, SPLIDAR_FUSED_1X=0): the same y in the same order, s summed in another order, so
    pi agrees to rounding (<= 1e-14 L1; 2e-12 if a count differs) and the iteration counts to +-1;
    relaunches are bit-identical."""
    f = random_flux(np.random.default_rng(4500 + n), n, 2)
    for dt in (torch.float64, torch.float32):
        P0 = spl.build_base(f, dt)
        T = np.array([[3.0, 61.5, 140.0, 250.0]])
        a = spl.Plan(P0, f.t_r, T, tol=1e-12)
        monkeypatch.setenv("SPLIDAR_FUSED_1X", "0")
        b = spl.Plan(P0, f.t_r, T, tol=1e-12)
        monkeypatch.delenv("SPLIDAR_FUSED_1X")
        assert a.fused and b.fused
        ia, ib = a.execute(check=False), b.execute(check=False)
        for v in range(T.shape[1]):
            assert abs(ia[v]["iters"] - ib[v]["iters"]) <= 1
            assert ia[v]["shift_l"] == ib[v]["shift_l"]
            # equal counts: rounding only; one more product: the last L1 change (< tol) on top
            bound = 1e-14 if ia[v]["iters"] == ib[v]["iters"] else 2e-12
            assert np.sum(np.abs(_np(a.pi[0, v]) - _np(b.pi[0, v]))) <= bound
        p1 = a.pi.clone()
        assert a.execute(check=False) == ia and torch.equal(a.pi, p1)
        a.close()
        b.close()


def test_ragged_large_n(spl):
    """N = 9001 (> 8192: the tiled flux-vector scans; a ragged last 512-column strip for the build and
    the graph-path GEMV; a 3-CTA cluster with a ragged last CTA for the structured solve): sampled rows
    of J_l P~0 vs the oracle's Eq. 4 rows, and pi from both solvers vs the long-double cross-check."""
    f = random_flux(np.random.default_rng(9001), 9001, 2)
    td = 157.25
    N = f.n_bins
    lam, F, Lam = oracle_vectors(f)
    v = spl.flux_vectors(f)
    assert np.max(np.abs(_np(v["F"]) - F)) <= 1e-13 * max(1.0, Lam)
    P0 = spl.build_base(f)
    l = oracle.shift_l(f, td)
    rows = [0, 1, 511, 512, 8999, 9000, l, (N - l) % N, 4500]
    want = sampled_rows(f, td, rows)
    got = np.stack([_np(P0[(r + l) % N]) for r in rows])
    assert np.max(np.abs(got - want)) <= TOL_E64
    pi, info = spl.stationary(P0, f.t_r, td)
    assert info["converged"]
    ref, _ = structured_pi(f, td, vectors=(lam, F, Lam))
    assert np.sum(np.abs(_np(pi) - ref)) <= TOL_PI64
    shape, S, B = spl.flux_items(f)
    pis, _ = spl.stationary_structured(shape, S, B, [td])
    assert np.sum(np.abs(_np(pis[0]) - ref)) <= TOL_PI64


def test_sweep_chunked_store_and_many_dead_times(spl):
    """splidar_sweep with n_store = 3 for 7 distinct (S, B) profiles (three rounds of builds) and 40
    dead times on one profile (two multi-vector passes of <= 32), N = 700 (fused solver) and 3000
    (graph path): every item vs its own single solve and a sample vs the oracle."""
    rng = np.random.default_rng(44)
    for N in (700, 3000):
        base = random_flux(rng, N, 1)
        shape = Flux(base.t_r, N, base.tau, base.sigma, (1.0,), 1.0)
        S = list(rng.uniform(0.1, 5.0, 6)) + [2.0] * 40
        B = list(rng.uniform(0.05, 1.5, 6)) + [0.7] * 40
        T = list(rng.uniform(0.0, 250.0, 6)) + list(np.linspace(1.0, 290.0, 40))
        pi, infos = spl.sweep(shape, S, B, T, n_store=3)
        got = _np(pi)
        for m in list(range(6)) + [6, 25, 45]:
            f = Flux(shape.t_r, N, shape.tau, shape.sigma, (S[m],), B[m])
            assert infos[m]["converged"] and infos[m]["shift_l"] == oracle.shift_l(f, T[m])
            P0 = spl.build_base(f)
            single, _ = spl.stationary(P0, f.t_r, T[m])
            assert np.sum(np.abs(got[m] - _np(single))) <= 1e-13, (N, m)
        for m in (0, 45):
            f = Flux(shape.t_r, N, shape.tau, shape.sigma, (S[m],), B[m])
            want = _oracle_pi(oracle.build_eq4(f, T[m]))
            assert np.sum(np.abs(got[m] - want)) <= TOL_PI64


@pytest.mark.parametrize("N", [700, 9001])
def test_sweep_matrix_free_equals_dense(spl, N):
    """splidar_sweep with P0_store = NULL (matrix-free: the structured operator) gives the dense sweep's
    pi (<= 1e-13 L1), the same shifts and Lambda, iterations +-1 (R25), for mixed (S, B, t_d) items
    including repeated profiles; N = 9001 takes cluster teams."""
    rng = np.random.default_rng(N)
    base = random_flux(rng, N, 2)
    shape = Flux(base.t_r, N, base.tau, base.sigma, (0.7, 0.3), 1.0)
    S = list(rng.uniform(0.1, 5.0, 5)) + [2.0] * 4
    B = list(rng.uniform(0.05, 1.5, 5)) + [0.7] * 4
    T = list(rng.uniform(0.0, 250.0, 5)) + [10.0, 75.0, 200.0, 310.0]
    pd, infd = spl.sweep(shape, S, B, T)
    pf, inff = spl.sweep(shape, S, B, T, matrix_free=True)
    for m in range(len(S)):
        assert inff[m]["converged"] and inff[m]["shift_l"] == infd[m]["shift_l"]
        assert abs(inff[m]["iters"] - infd[m]["iters"]) <= 1
        assert abs(inff[m]["lambda_total"] - infd[m]["lambda_total"]) <= 1e-13 * infd[m]["lambda_total"]
        assert np.sum(np.abs(_np(pf[m]) - _np(pd[m]))) <= 1e-13, m


@pytest.mark.parametrize("dtype,nv", [(torch.float64, 1), (torch.float64, 5), (torch.float32, 1)])
def test_eager_mode_equals_graph(spl, monkeypatch, dtype, nv):
    """SPLIDAR_EAGER=1 (host loop over the same kernels, for profilers) gives bit-identical pi and the same
    infos as the CUDA-graph plan: fp64 single vector (check fused into the GEMV), fp64 multi-vector and
    fp32 (separate check kernel); N = 3000 (graph path)."""
    f = random_flux(np.random.default_rng(3000 + nv), 3000, 2)
    tds = [float(x) for x in np.linspace(5.0, 280.0, nv)]
    P0 = spl.build_base(f, dtype)
    g = spl.Plan(P0, f.t_r, np.array([tds]), tol=1e-12)
    ig = g.execute(check=False)
    monkeypatch.setenv("SPLIDAR_EAGER", "1")
    e = spl.Plan(P0, f.t_r, np.array([tds]), tol=1e-12)
    monkeypatch.delenv("SPLIDAR_EAGER")
    ie = e.execute(check=False)
    assert torch.equal(g.pi, e.pi) and ig == ie
    g.close()
    e.close()


def test_max_size_dense(spl):
    """A matrix sized for the 180 GB of one B200: N = 110000 (ragged: not a multiple of 512), fp64,
    96.8 GB. Sampled rows of J_l P~0 vs the oracle's Eq. 4 rows, all row sums, and pi vs the
    long-double structured cross-check."""
    N = 110000
    ld = spl.leading_dim(N)
    need = N * ld * 8
    free, _ = torch.cuda.mem_get_info()
    if free < need + (6 << 30):
        pytest.skip(f"needs {need / 2**30:.0f} GiB free, have {free / 2**30:.0f}")
    f = Flux(100.0, N, (37.0, 71.0), (0.4, 0.9), (2.0, 0.6), 0.8)
    td = 142.5
    P0 = spl.build_base(f)
    l = oracle.shift_l(f, td)
    rows = [0, N - 1, l, (N - l) % N, 54321]
    want = sampled_rows(f, td, rows)
    got = np.stack([_np(P0[(r + l) % N]) for r in rows])
    assert np.max(np.abs(got - want)) <= TOL_E64
    rs = _np(P0.sum(dim=1, dtype=torch.float64))
    assert np.max(np.abs(rs - 1.0)) <= TOL_ROW
    pi, info = spl.stationary(P0, f.t_r, td)
    assert info["converged"]
    ref, _ = structured_pi(f, td)
    assert np.sum(np.abs(_np(pi) - ref)) <= TOL_PI64
    del P0
    torch.cuda.empty_cache()


def test_concurrent_streams_reentrant(spl):
    """The library is re-entrant for distinct (stream, workspace) pairs: a dense plan (graph path), a
    structured plan and a stored-matrix lambda_2 enqueued on three streams at once give bit-identical
    results to the same calls run one after another on the default stream."""
    f = random_flux(np.random.default_rng(77), 3000, 2)
    tds = [20.0, 140.0, 260.0]
    P0 = spl.build_base(f)
    shape, S, B = spl.flux_items(f)
    # sequential references
    plan = spl.Plan(P0, f.t_r, [tds])
    plan.execute()
    ref_dense = plan.pi.clone()
    plan.close()
    ref_struct, _ = spl.stationary_structured(shape, np.repeat(S, 3), np.repeat(B, 3), tds)
    ref_l2 = spl.second_eigenvalue_dense(P0, f.t_r, tds[0], ref_struct[0].contiguous())
    torch.cuda.synchronize()
    # concurrent: three streams, three workspaces
    s1, s2, s3 = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()
    torch.cuda.synchronize()
    with torch.cuda.stream(s1):
        p1 = spl.Plan(P0, f.t_r, [tds], stream=s1)
        p1.launch(stream=s1)
    with torch.cuda.stream(s2):
        sp = spl.StructPlan("solve", shape, np.repeat(S, 3), np.repeat(B, 3), tds, stream=s2)
        sp.launch(stream=s2)
    with torch.cuda.stream(s3):
        l2 = spl.second_eigenvalue_dense(P0, f.t_r, tds[0], ref_struct[0].contiguous(), stream=s3)
    p1.info(stream=s1)
    sp.info(stream=s2)
    torch.cuda.synchronize()
    assert torch.equal(p1.pi, ref_dense)
    assert torch.equal(sp.pi, ref_struct)
    assert l2 == ref_l2
    p1.close()
    sp.close()
