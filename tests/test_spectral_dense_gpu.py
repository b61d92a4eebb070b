"""f1 on a STORED matrix (splidar_second_eigenvalue_dense: the deflated 2-D subspace iteration of §4,
P:207-216, with every product one pass of the two-vector GEMV over P0) against:
  - the oracle's spectrum of the same matrix (oracle.second_eigenvalue = numpy eigvals of the rolled
    Eq. 4 matrix, or of a seeded generic row-stochastic matrix rolled by J_l);
  - the closed form of the S = 0 circulant (pin P5);
  - at sizes the dense oracle cannot reach (several dots chunks, config 5's N = 32768), the structured
    kernel's lambda_2 (independent arithmetic, itself pinned to the oracle in test_structured_gpu.py);
  - the degenerate rank-1 matrix (lambda_2 = 0) and fp32 storage."""
import math

import numpy as np
import pytest
import torch

import oracle
from workloads import Flux, config, parity_cases

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def spl():
    assert torch.cuda.is_available(), "GPU tests need a B200"
    from paper_2509_20500_b200 import build
    build.build()
    import paper_2509_20500_b200 as s
    return s


def _dense_lambda2(spl, P0, t_r, t_d, dtype_pi_tol=1e-12, **kw):
    pi, info = spl.stationary(P0, t_r, t_d, tol=dtype_pi_tol)
    assert info["converged"]
    return spl.second_eigenvalue_dense(P0, t_r, t_d, pi, **kw), pi


def _check(got, want, tol):
    assert got["converged"], got
    assert abs(got["modulus"] - abs(want)) <= tol, (got, want)
    if abs(want) > 1e-6:
        assert abs(got["phase"] - math.atan2(want.imag, want.real)) <= tol / abs(want) + 1e-9, (got, want)
    assert abs(got["gap"] - (1 - abs(want))) <= tol


CASES = [c for c in parity_cases() if 4 <= c.flux.n_bins <= 1100] + [config(1).items[0]]


@pytest.mark.parametrize("case", CASES, ids=[f"N{c.flux.n_bins}-td{c.t_d:.1f}" for c in CASES])
def test_dense_lambda2_vs_oracle(spl, case):
    f = case.flux
    P0 = spl.build_base(f, torch.float64)
    got, _ = _dense_lambda2(spl, P0, f.t_r, case.t_d)
    want = oracle.second_eigenvalue(oracle.build_eq4(f, case.t_d))
    _check(got, want, 1e-8)


def _generic(n, seed):
    """Seeded row-stochastic matrix with a well-separated complex lambda_2 pair: from state i, mass
    0.8 goes to the states of group (i + 1) mod 3 (random weights), 0.2 anywhere (random weights);
    the lumped 3-group chain contributes ~0.8 e^{+-2 pi i / 3}, the random rest ~1 / sqrt(n)."""
    rng = np.random.default_rng(seed)
    g = np.arange(n) % 3
    R1 = rng.random((n, n)) * (g[None, :] == (g[:, None] + 1) % 3)
    R2 = rng.random((n, n))
    return 0.8 * R1 / R1.sum(axis=1, keepdims=True) + 0.2 * R2 / R2.sum(axis=1, keepdims=True)


@pytest.mark.parametrize("n,td", [(500, 0.0), (777, 37.0), (1023, 250.0)])
def test_dense_lambda2_generic_matrix(spl, n, td):
    P = _generic(n, n)
    P0 = spl.empty_matrix(n, torch.float64)
    P0.copy_(torch.from_numpy(P))
    t_r = 100.0
    l = spl.shift(t_r, n, td)
    got, _ = _dense_lambda2(spl, P0, t_r, td)
    want = oracle.second_eigenvalue(np.roll(P, -l, axis=0))   # row i of J_l P0 = row (i + l) of P0
    _check(got, want, 1e-9)
    if l % 3 == 0:   # the group cycle survives the shift: a complex pair ~0.8 e^{2 pi i / 3}
        assert abs(want.imag) > 0.5


def test_dense_lambda2_fp32_storage(spl):
    f = config(1).items[0].flux
    td = config(1).items[0].t_d
    P0 = spl.build_base(f, torch.float32)
    got, _ = _dense_lambda2(spl, P0, f.t_r, td)
    # the same fp32 entries widened to fp64 on the host: the iteration's own error is what is measured
    # (rows sum to 1 only to fp32 rounding; the Perron root rho ~ 1 +- 1e-7 is deflated with pi either way)
    P = P0.double().cpu().numpy()
    l = spl.shift(f.t_r, f.n_bins, td)
    want = oracle.second_eigenvalue(np.roll(P, -l, axis=0))
    _check(got, want, 1e-7)


@pytest.mark.parametrize("B,N,td", [(1.0, 256, 75.0), (10.0, 33, 250.0), (0.5, 2048, 10.0)])
def test_dense_lambda2_circulant_closed_form(spl, B, N, td):
    """S = 0: lambda_2 = w^l (1 - r) / (1 - r w), w = e^{2 pi i / N}, r = e^{-B / N} (pin P5)."""
    f = Flux(100.0, N, (50.0,), (1.0,), (0.0,), B)
    P0 = spl.build_base(f, torch.float64)
    pi = torch.full((N,), 1.0 / N, dtype=torch.float64, device="cuda")
    got = spl.second_eigenvalue_dense(P0, 100.0, td, pi)
    l = spl.shift(100.0, N, td)
    r = math.exp(-B / N)
    w = np.exp(2j * np.pi / N)
    mu = w ** l * (1 - r) / (1 - r * w)
    assert got["converged"]
    assert abs(got["modulus"] - abs(mu)) <= 1e-9
    assert abs(got["phase"] - abs(np.angle(mu))) <= 1e-8


@pytest.mark.parametrize("k", [4, 5])
def test_dense_equals_structured_large(spl, k):
    """N = 16384 / 32768 (configs 4, 5; 32 / 64 dots chunks, ragged GEMV pieces): the stored-matrix
    lambda_2 equals the structured kernel's to far below the paper's reported precision."""
    it = config(k).items[0]
    f = it.flux
    P0 = spl.build_base(f, torch.float64)
    got, pi = _dense_lambda2(spl, P0, f.t_r, it.t_d)
    shape, S, B = spl.flux_items(f)
    ref = spl.second_eigenvalue(shape, S, B, [it.t_d], pi.reshape(1, -1).contiguous())[0]
    assert got["converged"] and ref["converged"]
    assert abs(spl.lambda2_of(ref) - got["lambda2"]) <= 1e-10, (got, ref)


def test_dense_ragged_multi_chunk(spl):
    """N = 9001 (18 dots chunks and 18 GEMV strips, the last of each ragged) vs structured."""
    rng = np.random.default_rng(5)
    f = Flux(100.0, 9001, (40.0, 63.0), (0.5, 1.5), (0.8, 0.4), 0.6)
    td = float(rng.uniform(0, 300))
    P0 = spl.build_base(f, torch.float64)
    got, pi = _dense_lambda2(spl, P0, f.t_r, td)
    shape, S, B = spl.flux_items(f)
    ref = spl.second_eigenvalue(shape, S, B, [td], pi.reshape(1, -1).contiguous())[0]
    assert abs(spl.lambda2_of(ref) - got["lambda2"]) <= 1e-10, (got, ref)


def test_dense_rank_one_matrix(spl):
    """Every row equal to p: P~ = 1 p, A = P~ - 1 pi = 0, lambda_2 = 0 for any shift."""
    n = 700
    p = np.random.default_rng(3).random(n) + 0.1
    p /= p.sum()
    P0 = spl.empty_matrix(n, torch.float64)
    P0.copy_(torch.from_numpy(np.tile(p, (n, 1))))
    pi = torch.from_numpy(p).cuda()
    got = spl.second_eigenvalue_dense(P0, 100.0, 30.0, pi)
    assert got["converged"] and got["modulus"] <= 1e-12 and got["iters"] <= 3


def test_dense_lambda2_deterministic_and_noconv(spl):
    f = config(1).items[0].flux
    P0 = spl.build_base(f, torch.float64)
    a, pi = _dense_lambda2(spl, P0, f.t_r, 75.0)
    b = spl.second_eigenvalue_dense(P0, f.t_r, 75.0, pi)
    assert a == b
    c = spl.second_eigenvalue_dense(P0, f.t_r, 75.0, pi, max_iter=2, check=False)
    assert not c["converged"] and c["iters"] == 2
    with pytest.raises(spl.SplidarError):
        spl.second_eigenvalue_dense(P0, f.t_r, 75.0, pi, max_iter=2)


def test_dense_equals_structured_max_n(spl):
    """N = 65536 (a 34 GB fp64 matrix; the structured lambda_2 on a 16-CTA cluster, its largest team):
    the two independent lambda_2 computations agree."""
    f = Flux(100.0, 65536, (30.0, 70.0), (0.05, 0.2), (1.5, 0.7), 0.9)
    td = 123.4
    shape, S, B = spl.flux_items(f)
    pi, _ = spl.stationary_structured(shape, S, B, [td])
    ref = spl.second_eigenvalue(shape, S, B, [td], pi)[0]
    P0 = spl.build_base(f)
    got = spl.second_eigenvalue_dense(P0, f.t_r, td, pi[0].contiguous())
    del P0
    torch.cuda.empty_cache()
    assert got["converged"] and ref["converged"]
    assert abs(spl.lambda2_of(ref) - got["lambda2"]) <= 1e-10, (got, ref)
