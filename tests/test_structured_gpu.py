"""SURVEY §8(f) rows f2 (matrix-free stationary solve) and f1 (second eigenvalue, mixing steps, bin
trajectories) on the GPU, through the C ABI, against the CPU oracle (pytest -m gpu).

The structured operator computes x^T P~0 from one prefix scan (§3.4) and never stores the
matrix; the oracle builds P~ entry by entry from Eq. 4, solves pi densely and takes the
spectrum with numpy.linalg.eigvals. Tolerances: pi <= 1e-10 L1 (BASELINE.json), lambda_2 <= 1e-8 in
modulus and phase (SPEC second_eigenvalue), mixing steps exact (integers decided in fp64 on both
sides), trajectories <= 1e-13.
"""
import math

import numpy as np
import pytest
import torch

import oracle
from workloads import Flux, config, parity_cases, random_flux

from ._structured import oracle_vectors, structured_pi

pytestmark = pytest.mark.gpu

TOL_PI64 = 1e-10


@pytest.fixture(scope="module")
def spl():
    assert torch.cuda.is_available(), "GPU tests need a B200"
    from paper_2509_20500_b200 import build
    build.build()
    import paper_2509_20500_b200 as s
    return s


def _np(t):
    return t.detach().cpu().numpy()


def _one(spl, flux, t_d, **kw):
    shape, S, B = spl.flux_items(flux)
    pi, infos = spl.stationary_structured(shape, S, B, [t_d], **kw)
    return pi[0], infos[0]


CASES = parity_cases()
IDS = [f"N{c.flux.n_bins}-K{c.flux.n_pulses}-td{c.t_d:.2f}" for c in CASES]


# ------------------------------------------------------------- f2: stationary solve
@pytest.mark.parametrize("case", CASES, ids=IDS)
def test_structured_pi_vs_oracle(spl, case):
    f = case.flux
    pi, info = _one(spl, f, case.t_d)
    assert info["converged"] and info["l1_change"] < 1e-12
    assert info["shift_l"] == oracle.shift_l(f, case.t_d)
    assert abs(info["lambda_total"] - oracle.Lambda(f)) <= 1e-13 * max(1.0, oracle.Lambda(f))
    want = oracle.stationary_dense(oracle.build_eq4(f, case.t_d))
    got = _np(pi)
    assert np.sum(np.abs(got - want)) <= TOL_PI64
    assert abs(got.sum() - 1.0) <= 1e-13 and np.all(got > 0)


@pytest.mark.parametrize("case", CASES[::2], ids=IDS[::2])
def test_structured_equals_dense_path(spl, case):
    """Same pi and the same iteration count as the dense GEMV solve of the stored P~0."""
    f = case.flux
    pi_s, info_s = _one(spl, f, case.t_d)
    P0 = spl.build_base(f)
    pi_d, info_d = spl.stationary(P0, f.t_r, case.t_d)
    assert np.sum(np.abs(_np(pi_s) - _np(pi_d))) <= 1e-13
    assert abs(info_s["iters"] - info_d["iters"]) <= 1


def test_structured_batched_items_and_noconv(spl):
    """A batch of items with shared and distinct (S, B) and several dead times, in one launch; an
    item capped at max_iter = 2 reports ENOCONV with the second iterate."""
    rng = np.random.default_rng(11)
    base = random_flux(rng, 1537, 2)
    shape = Flux(base.t_r, base.n_bins, base.tau, base.sigma, (0.7, 0.3), 1.0)
    S = np.array([0.5, 0.5, 3.0, 3.0, 8.0, 0.01])
    B = np.array([0.2, 0.2, 1.0, 1.0, 0.05, 1.5])
    T = np.array([0.0, 57.0, 133.3, 20.0, 250.0, 99.0])
    pi, infos = spl.stationary_structured(shape, S, B, T)
    for m in range(6):
        f = Flux(shape.t_r, shape.n_bins, shape.tau, shape.sigma, tuple(S[m] * np.array(shape.signal)), B[m])
        want = oracle.stationary_dense(oracle.build_eq4(f, T[m]))
        assert np.sum(np.abs(_np(pi[m]) - want)) <= TOL_PI64, m
        assert infos[m]["converged"]
    with pytest.raises(spl.SplidarError) as e:
        spl.stationary_structured(shape, S[:1], B[:1], T[1:2], max_iter=2)
    assert e.value.status == spl.ENOCONV
    pi2, inf2 = spl.stationary_structured(shape, S[:1], B[:1], T[1:2], max_iter=2, check=False)
    f = Flux(shape.t_r, shape.n_bins, shape.tau, shape.sigma, tuple(S[0] * np.array(shape.signal)), B[0])
    P = oracle.build_eq4(f, T[1])
    x = np.full(f.n_bins, 1.0 / f.n_bins)
    for _ in range(2):
        x = x @ P
        x /= x.sum()
    assert inf2[0]["iters"] == 2 and not inf2[0]["converged"]
    assert np.sum(np.abs(_np(pi2[0]) - x)) <= 1e-13


def test_structured_config3_all_items(spl):
    w = config(3)
    base = w.items[0].flux
    shape = Flux(base.t_r, base.n_bins, base.tau, base.sigma, (1.0,), 1.0)
    S = np.array([it.flux.signal[0] for it in w.items])
    B = np.array([it.flux.background for it in w.items])
    T = np.array([it.t_d for it in w.items])
    pi, infos = spl.stationary_structured(shape, S, B, T)
    got = _np(pi)
    for m, it in enumerate(w.items):
        assert infos[m]["converged"]
        ref, _ = structured_pi(it.flux, it.t_d)
        assert np.sum(np.abs(got[m] - ref)) <= TOL_PI64, m
    for m in (0, 42):
        it = w.items[m]
        want, _, _, ok = oracle.stationary_power(oracle.build_eq4(it.flux, it.t_d), 1e-15)
        assert np.sum(np.abs(got[m] - want)) <= TOL_PI64


@pytest.mark.parametrize("k", [4, 5])
def test_structured_full_size_configs(spl, k):
    """Configs 4-5 (N = 16384 / 32768: clusters of 4 / 8 CTAs) incl. config 5's 16-value sweep, vs the
    long-double structured cross-check and the oracle's streamed Eq. 4 residual."""
    w = config(k)
    f = w.items[0].flux
    tds = [w.items[0].t_d] + [it.t_d for it in w.sweep]
    shape, S, B = spl.flux_items(f)
    pi, infos = spl.stationary_structured(shape, np.repeat(S, len(tds)), np.repeat(B, len(tds)), tds)
    vec = oracle_vectors(f)
    for v, td in enumerate(tds):
        ref, _ = structured_pi(f, td, vectors=vec)
        assert np.sum(np.abs(_np(pi[v]) - ref)) <= TOL_PI64, td
        assert infos[v]["shift_l"] == oracle.shift_l(f, td)
    if k == 4:
        y = oracle.left_matvec_streamed(f, tds[0], _np(pi[0]))
        assert np.sum(np.abs(y - _np(pi[0]))) <= 1e-11


def test_structured_max_n_cluster16(spl):
    """N = 65536: a non-portable cluster of 16 CTAs (the largest N the structured path takes)."""
    f = Flux(100.0, 65536, (30.0, 70.0), (0.05, 0.2), (1.5, 0.7), 0.9)
    pi, info = _one(spl, f, 123.4)
    ref, _ = structured_pi(f, 123.4)
    assert info["converged"]
    assert np.sum(np.abs(_np(pi) - ref)) <= TOL_PI64
    with pytest.raises(spl.SplidarError):
        spl.structured_workspace(65537 * 2)


def test_structured_constant_flux(spl):
    f = Flux(100.0, 1000, (50.0,), (1.0,), (0.0,), 3.0)
    pi, info = _one(spl, f, 75.0)
    assert np.max(np.abs(_np(pi) - 1e-3)) <= 1e-15 and info["iters"] <= 2


def test_structured_deterministic(spl):
    f = config(5).items[0].flux
    a, _ = _one(spl, f, 430.0)
    b, _ = _one(spl, f, 430.0)
    assert torch.equal(a, b)


# ------------------------------------------------------------- f1: second eigenvalue
SPEC_CASES = [c for c in CASES if 4 <= c.flux.n_bins <= 1100] + [config(1).items[0]]


def _lambda2(spl, flux, t_d, pi):
    shape, S, B = spl.flux_items(flux)
    return spl.second_eigenvalue(shape, S, B, [t_d], pi.reshape(1, -1).contiguous())[0]


@pytest.mark.parametrize("case", SPEC_CASES, ids=[f"N{c.flux.n_bins}-td{c.t_d:.1f}" for c in SPEC_CASES])
def test_lambda2_vs_oracle(spl, case):
    f = case.flux
    pi, _ = _one(spl, f, case.t_d)
    got = _lambda2(spl, f, case.t_d, pi)
    P = oracle.build_eq4(f, case.t_d)
    want = oracle.second_eigenvalue(P)
    assert got["converged"]
    assert abs(got["modulus"] - abs(want)) <= 1e-8
    if abs(want) > 1e-6:
        assert abs(got["phase"] - math.atan2(want.imag, want.real)) <= 1e-8 / abs(want) + 1e-9
    assert abs(got["gap"] - (1 - abs(want))) <= 1e-8


@pytest.mark.parametrize("B,N,td", [(1.0, 256, 75.0), (3.0, 50, 75.0), (10.0, 33, 250.0), (0.5, 4096, 10.0)])
def test_lambda2_circulant_closed_form(spl, B, N, td):
    """S = 0: lambda_2 = w^l (1 - r) / (1 - r w), w = e^{2 pi i / N} (pin P5 / f1 circulant)."""
    f = Flux(100.0, N, (50.0,), (1.0,), (0.0,), B)
    pi = torch.full((N,), 1.0 / N, dtype=torch.float64, device="cuda")
    got = _lambda2(spl, f, td, pi)
    l = spl.shift(100.0, N, td)
    r = math.exp(-B / N)
    w = np.exp(2j * np.pi / N)
    mu = w ** l * (1 - r) / (1 - r * w)
    assert abs(got["modulus"] - abs(mu)) <= 1e-9
    assert abs(got["phase"] - abs(np.angle(mu))) <= 1e-8


def test_lambda2_large_n_vs_trajectory(spl):
    """Config 4 (N = 16384): no dense spectrum; lambda_2 is checked against the dynamics it fixes:
    the deviation of a bin trajectory from pi fits Re(c lambda_2^n) over a tail window."""
    it = config(4).items[0]
    f = it.flux
    pi, _ = _one(spl, f, it.t_d)
    got = _lambda2(spl, f, it.t_d, pi)
    assert got["converged"] and 0 < got["modulus"] < 1
    lam = spl.lambda2_of(got)
    start = torch.zeros(f.n_bins, dtype=torch.float64, device="cuda")
    start[100] = 1.0
    bin_ = int(torch.argmax(pi))
    n1 = int(math.log(1e-9) / math.log(got["modulus"]))   # residual still >> rounding at n1
    n0 = n1 // 2
    assert n1 - n0 >= 6
    tr, _ = spl.bin_trajectory(f, it.t_d, start, bin_, n1)
    r = _np(tr)[n0:n1 + 1] - float(pi[bin_])
    n = np.arange(n0, n1 + 1)
    A = np.stack([(lam ** n).real, -(lam ** n).imag], axis=1) if lam.imag > 0 else (lam.real ** n)[:, None]

    def fit_err(A):
        coef, *_ = np.linalg.lstsq(A, r, rcond=None)
        return np.max(np.abs(A @ coef - r)) / np.max(np.abs(r))
    good = fit_err(A)
    lb = lam * 1.05
    bad = fit_err(np.stack([(lb ** n).real, -(lb ** n).imag], axis=1) if lam.imag > 0 else (lb.real ** n)[:, None])
    assert good <= 1e-2 and bad > 3 * good, (got, good, bad)


# ------------------------------------------------------------- f1: mixing steps, trajectories
MIX_CASES = [(Flux(100.0, 128, (40.0,), (0.8,), (2.0,), B), 75.0) for B in (0.1, 3.0, 6.0)] + \
            [(c.flux, c.t_d) for c in CASES if c.flux.n_bins in (64, 255)] + [(config(1).items[0].flux, 75.0)]


@pytest.mark.parametrize("f,td", MIX_CASES, ids=[f"N{f.n_bins}-B{f.background:.2f}-td{td:.1f}" for f, td in MIX_CASES])
def test_mixing_steps_vs_oracle(spl, f, td):
    P = oracle.build_eq4(f, td)
    pi_o = oracle.stationary_dense(P)
    pi, _ = _one(spl, f, td, tol=1e-14)
    n_gpu, per = spl.mixing_steps(f, td, pi, eps=1e-3)
    n_or, first = oracle.mixing_steps(P, pi_o, 1e-3)
    assert n_gpu == n_or
    assert np.array_equal(_np(per), first)


def test_mixing_steps_large(spl):
    """N = 4096 (4096 starts, one CTA each): per-start counts against the oracle on sampled rows via
    the oracle's own products (Eq. 4 rows, power by repeated row-vector products)."""
    it = config(3).items[7]
    f = it.flux
    pi, _ = _one(spl, f, it.t_d, tol=1e-14)
    n_gpu, per = spl.mixing_steps(f, it.t_d, pi, eps=1e-3)
    per = _np(per)
    assert n_gpu == per.max() and np.all(per >= 1)
    # three starts: the first n with TV <= eps from the oracle's matrix rows (streamed products)
    P = oracle.build_eq4(f, it.t_d)
    pi_np = _np(pi)
    for i in (0, 1234, int(np.argmax(per))):
        v = np.zeros(f.n_bins)
        v[i] = 1.0
        n = 0
        while True:
            v = v @ P
            n += 1
            if 0.5 * np.abs(v - pi_np).sum() <= 1e-3:
                break
        assert per[i] == n, i


@pytest.mark.parametrize("f,td", MIX_CASES[:4], ids=[f"N{f.n_bins}-{td:.0f}" for f, td in MIX_CASES[:4]])
def test_bin_trajectory_vs_oracle(spl, f, td):
    rng = np.random.default_rng(f.n_bins)
    start = rng.random(f.n_bins)
    start /= start.sum()
    P = oracle.build_eq4(f, td)
    bin_ = int(rng.integers(0, f.n_bins))
    want, want_v = oracle.bin_trajectory(P, start, bin_, 40)
    tr, fin = spl.bin_trajectory(f, td, torch.tensor(start, device="cuda"), bin_, 40)
    assert np.max(np.abs(_np(tr) - want)) <= 1e-13
    assert np.max(np.abs(_np(fin) - want_v)) <= 1e-13
    tr0, fin0 = spl.bin_trajectory(f, td, torch.tensor(start, device="cuda"), bin_, 0)
    assert _np(tr0)[0] == start[bin_] and np.array_equal(_np(fin0), start)


# ------------------------------------------------------------- extreme flux (Lambda near the 600 guard)
@pytest.mark.parametrize("S,B,N", [(450.0, 120.0, 512), (0.0, 590.0, 300), (30.0, 1e-6, 1024)],
                         ids=["Lambda570", "const590", "tinyB"])
def test_extreme_flux_all_paths(spl, S, B, N):
    """Lambda = 570 / 590 (e^{-Lambda} ~ 1e-250: the factored entries span ~250 decades) and a vanishing
    floor B = 1e-6: the dense fused path, the dense graph path and the structured path all match the
    oracle's Eq. 4 pi."""
    f = Flux(100.0, N, (42.0,), (0.7,), (S,), B)
    td = 63.3
    want = oracle.stationary_dense(oracle.build_eq4(f, td))
    P0 = spl.build_base(f)
    got_e = _np(P0)
    assert np.max(np.abs(got_e - oracle.build_eq4(f, 0.0))) <= 1e-12
    pi_d, info = spl.stationary(P0, f.t_r, td, max_iter=10 ** 6)
    assert np.sum(np.abs(_np(pi_d) - want)) <= TOL_PI64
    pi_s, _ = _one(spl, f, td, max_iter=10 ** 6)
    assert np.sum(np.abs(_np(pi_s) - want)) <= TOL_PI64


def test_extreme_flux_rejected_beyond_guard(spl):
    f = Flux(100.0, 256, (42.0,), (0.7,), (500.0,), 101.0)      # Lambda = 601 > 600 (reading R15)
    with pytest.raises(spl.SplidarError):
        spl.build_base(f)
    with pytest.raises(spl.SplidarError):
        _one(spl, f, 10.0)


def test_mixing_steps_cluster_team(spl):
    """N = 6000 (> 4096: a 2-CTA cluster per start bin, DSMEM pushes): per-start first hits of three
    starts against repeated products with the oracle's Eq. 4 matrix."""
    f = random_flux(np.random.default_rng(6000), 6000, 2)
    td = 71.0
    pi, _ = _one(spl, f, td, tol=1e-14)
    n_gpu, per = spl.mixing_steps(f, td, pi, eps=1e-3)
    per = _np(per)
    assert n_gpu == per.max() and np.all(per >= 1)
    P = oracle.build_eq4(f, td)
    pi_np = _np(pi)
    for i in (0, 2999, int(np.argmax(per))):
        v = np.zeros(f.n_bins)
        v[i] = 1.0
        n = 0
        while True:
            v = v @ P
            n += 1
            if 0.5 * np.abs(v - pi_np).sum() <= 1e-3:
                break
        assert per[i] == n, i


@pytest.mark.parametrize("N", [255, 256, 257, 4095, 4096, 4097, 8191, 8192, 8193, 12289])
def test_team_boundaries(spl, N):
    """Each side of every team-shape boundary (warp <= 256 < CTA <= 4096 < cluster; cluster size steps
    every 4096 bins): the structured pi equals the dense GEMV path's pi, and lambda_2 the oracle's."""
    f = random_flux(np.random.default_rng(N), N, 2)
    td = float(np.random.default_rng(N + 1).uniform(0.0, 3.0 * f.t_r))
    pi_s, info_s = _one(spl, f, td)
    P0 = spl.build_base(f)
    pi_d, info_d = spl.stationary(P0, f.t_r, td)
    assert info_s["converged"] and abs(int(info_s["iters"]) - info_d["iters"]) <= 1
    assert np.sum(np.abs(_np(pi_s) - _np(pi_d))) <= 1e-13
    del P0
    if N <= 4097:
        got = _lambda2(spl, f, td, pi_s)
        want = oracle.second_eigenvalue(oracle.build_eq4(f, td))
        assert got["converged"] and abs(got["modulus"] - abs(want)) <= 1e-8


@pytest.mark.parametrize("N", [12289, 32768])
def test_cluster_shift_edges(spl, N):
    """Cluster teams at the shifts where the pushes' destination runs change shape: l = 0 (every CTA
    pushes to itself), l = 1, l at and next to a chunk boundary (2048 at 4 bins per thread, 4096 at 8),
    l = N - 1 (wrap of all but one position); N = 12289 leaves a last CTA of 1 position. One item
    (4 bins per thread, one cluster) and 17 items (8 bins per thread, two waves) against the dense GEMV
    path's pi for the same P~0."""
    f = random_flux(np.random.default_rng(N + 7), N, 2)
    ls = [0, 1, 2047, 2048, 4095, 4096, N - 1]
    tds = [0.0 if l == 0 else (l - 0.5) * f.t_r / N for l in ls]
    assert [spl.shift(f.t_r, N, t) for t in tds] == ls
    P0 = spl.build_base(f)
    pis_d, infos_d = [], []
    for td in tds:
        p, i = spl.stationary(P0, f.t_r, td)
        pis_d.append(_np(p))
        infos_d.append(i)
    del P0
    shape, S, B = spl.flux_items(f)
    for td, want, inf_d in zip(tds, pis_d, infos_d):                     # one item: E = 4
        got, inf = _one(spl, f, td)
        assert inf["converged"] and abs(int(inf["iters"]) - inf_d["iters"]) <= 1
        assert np.sum(np.abs(_np(got) - want)) <= 1e-13, td
    T = (tds * 3)[:17]                                                   # 17 items: E = 8, two waves
    pis, infos = spl.stationary_structured(shape, np.repeat(S, 17), np.repeat(B, 17), T)
    for m in range(17):
        k = m % len(tds)
        assert bool(infos[m]["converged"])
        assert np.sum(np.abs(_np(pis[m]) - pis_d[k])) <= 1e-13, (m, ls[k])


@pytest.mark.parametrize("kind", ["solve", "lambda2"])
def test_plan_graph_replay_equals_eager(spl, kind):
    """A structured plan's first launch is eager, later ones replay a captured CUDA graph: identical
    results (bitwise), iteration counts and a positive kernel time from the graph's event nodes."""
    it = config(4).items[0]
    shape, S, B = spl.flux_items(it.flux)
    T = [it.t_d, 75.0, 430.0]
    S3, B3 = np.repeat(S, 3), np.repeat(B, 3)
    pi = None
    if kind == "lambda2":
        pi, _ = spl.stationary_structured(shape, S3, B3, T)
    plan = spl.StructPlan(kind, shape, S3, B3, T, pi=pi)
    outs = []
    for _ in range(3):
        plan.launch()
        infos, ms = plan.info()
        assert ms > 0.0
        outs.append((plan.pi.clone() if kind == "solve" else None, infos.copy()))
    plan.close()
    for o in outs[1:]:
        if kind == "solve":
            assert torch.equal(o[0], outs[0][0])
        assert np.array_equal(o[1], outs[0][1])
