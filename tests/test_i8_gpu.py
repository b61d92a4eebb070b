"""The int8 tensor-core GEMV (power_i8.cu: tcgen05.mma kind::i8, exact split of P~0 into u8 planes
with a per-column exponent and of x into 7 u8 slices) against the FP64 GEMV on the same plans, and
through the same plans against the oracle.

The split is exact for P~0 (every fp32 / fp64 entry is an integer multiple of its column's scale,
pinned by the range test) and truncates x at 2^-56 of its largest entry, so y agrees with the FP64
GEMV to ~1e-15 relative and pi to the same level; iteration counts are equal or +-1 (the stop test
compares an L1 change with 1e-12). A matrix that fails the range test must run the FP64 kernel.
"""
import os

import numpy as np
import pytest
import torch

import oracle
from workloads import Flux, config, random_flux

from ._structured import structured_pi

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def spl():
    assert torch.cuda.is_available(), "GPU tests need a B200"
    from paper_2509_20500_b200 import build
    build.build()
    import paper_2509_20500_b200 as s
    return s


def _solve(spl, P0, t_r, tds, env, monkeypatch, tol=1e-12):
    monkeypatch.setenv("SPLIDAR_I8", env)
    monkeypatch.setenv("SPLIDAR_FUSED", "0")         # N <= 2048 would take the fused small-N solver
    plan = spl.Plan(P0, t_r, np.array(tds).reshape(P0.shape[0] if P0.dim() == 3 else 1, -1), tol=tol)
    infos = plan.execute(check=False)
    kind = plan.gemv()
    pi = plan.pi.detach().cpu().numpy().copy()
    plan.close()
    return pi, infos, kind


def _c5_flux(N):
    f0 = config(5).items[0].flux
    return Flux(f0.t_r, N, f0.tau, f0.sigma, f0.signal, f0.background)


@pytest.mark.parametrize("N,V,dtype,env", [(1024, 8, torch.float32, "1"), (4096, 17, torch.float32, "1"),
                                           (6144, 18, torch.float32, "1"), (4096, 16, torch.float64, "2"),
                                           (2176, 9, torch.float64, "2")])
def test_i8_equals_fp64_gemv(spl, monkeypatch, N, V, dtype, env):
    f = _c5_flux(N)
    w = config(5)
    tds = ([w.items[0].t_d] + [it.t_d for it in w.sweep] + [333.3])[:V]
    P0 = spl.build_base(f, dtype)
    pi8, inf8, k8 = _solve(spl, P0, f.t_r, tds, env, monkeypatch)
    pif, inff, kf = _solve(spl, P0, f.t_r, tds, "0", monkeypatch)
    assert k8 == "tensor_i8" and kf == "fp64"
    assert all(i["converged"] for i in inf8)
    assert np.max(np.sum(np.abs(pi8 - pif), axis=-1)) <= 1e-13
    for a, b in zip(inf8, inff):
        assert abs(a["iters"] - b["iters"]) <= 1
    # and against the oracle's own Eq. 4 rows for two of the dead times (pi P~ = pi)
    if N <= 4096:
        for v in (0, V - 1):
            y = oracle.left_matvec_streamed(f, tds[v], pi8[0, v])
            tol = 1e-11 if dtype == torch.float64 else 1e-5
            assert np.sum(np.abs(y - pi8[0, v])) <= tol


def test_i8_batched_matrices(spl, monkeypatch):
    """M = 3 matrices x 8 dead times (active-matrix list, per-matrix column exponents). Lambda <= 4
    keeps every column within e^Lambda < 2^8 of its maximum (the range of 4 fp32 planes); larger
    fluxes take the FP64 kernel (test_i8_range_test_falls_back)."""
    rng = np.random.default_rng(88)
    fl = [random_flux(rng, 2048, 2, sigma_bins=(1, 10), s_range=(0.5, 1.5), b_range=(0.2, 1.0)) for _ in range(3)]
    fl = [Flux(100.0, 2048, f.tau, f.sigma, f.signal, f.background) for f in fl]
    P0 = spl.build_base_batched(fl, torch.float32)
    tds = rng.uniform(0, 300, (3, 8))
    pi8, inf8, k8 = _solve(spl, P0, 100.0, tds, "1", monkeypatch)
    pif, inff, kf = _solve(spl, P0, 100.0, tds, "0", monkeypatch)
    assert k8 == "tensor_i8"
    assert np.max(np.sum(np.abs(pi8 - pif), axis=-1)) <= 1e-13
    for m in range(3):
        ref, _ = structured_pi(fl[m], tds[m, 0])
        assert np.sum(np.abs(pi8[m, 0] - ref)) <= 1e-5      # fp32 storage tolerance


def test_i8_deterministic(spl, monkeypatch):
    f = _c5_flux(4096)
    tds = [10.0 + 30 * k for k in range(17)]
    P0 = spl.build_base(f, torch.float32)
    a, _, _ = _solve(spl, P0, f.t_r, tds, "1", monkeypatch)
    b, _, _ = _solve(spl, P0, f.t_r, tds, "1", monkeypatch)
    assert np.array_equal(a, b)


def test_i8_range_test_falls_back(spl, monkeypatch):
    """A row-stochastic matrix with one column spanning 2^12 (beyond the 2^8 of 4 fp32 planes) must
    run the FP64 kernel -- and give its exact result; with the range restored the int8 kernel runs."""
    N = 2048
    rng = np.random.default_rng(5)
    A = rng.uniform(0.5, 1.0, (N, N))
    A[:, 7] = np.where(np.arange(N) % 2 == 0, 1.0, 2.0 ** -12)
    A /= A.sum(axis=1, keepdims=True)
    P0 = spl.empty_matrix(N, torch.float32)
    P0.copy_(torch.from_numpy(A.astype(np.float32)))
    tds = [float(t) for t in rng.uniform(0, 100, 8)]
    pi8, _, k8 = _solve(spl, P0, 100.0, tds, "1", monkeypatch)
    pif, _, kf = _solve(spl, P0, 100.0, tds, "0", monkeypatch)
    assert k8 == "fp64" and np.array_equal(pi8, pif)
    B = rng.uniform(0.5, 1.0, (N, N))
    B /= B.sum(axis=1, keepdims=True)
    P0.copy_(torch.from_numpy(B.astype(np.float32)))
    pi8, _, k8 = _solve(spl, P0, 100.0, tds, "1", monkeypatch)
    pif, _, _ = _solve(spl, P0, 100.0, tds, "0", monkeypatch)
    assert k8 == "tensor_i8"
    assert np.max(np.sum(np.abs(pi8 - pif), axis=-1)) <= 1e-13


def test_i8_zero_columns(spl, monkeypatch):
    """All-zero columns (E_j = the largest exponent, every shift negative) and exact zeros elsewhere."""
    N = 1024
    rng = np.random.default_rng(6)
    A = rng.uniform(0.5, 1.0, (N, N))
    A[:, 100:116] = 0.0
    A[rng.uniform(size=(N, N)) < 0.05] = 0.0
    A /= A.sum(axis=1, keepdims=True)
    P0 = spl.empty_matrix(N, torch.float32)
    P0.copy_(torch.from_numpy(A.astype(np.float32)))
    tds = [float(t) for t in rng.uniform(0, 100, 8)]
    pi8, _, k8 = _solve(spl, P0, 100.0, tds, "1", monkeypatch)
    pif, _, _ = _solve(spl, P0, 100.0, tds, "0", monkeypatch)
    assert k8 == "tensor_i8"
    assert np.all(pi8[0, :, 100:116] == 0.0)
    assert np.max(np.sum(np.abs(pi8 - pif), axis=-1)) <= 1e-13


def test_i8_not_used_where_unsupported(spl, monkeypatch):
    f = _c5_flux(4096)
    P0 = spl.build_base(f, torch.float32)
    _, _, k = _solve(spl, P0, f.t_r, [10.0, 20.0], "1", monkeypatch)          # V < 8
    assert k == "fp64"
    P0d = spl.build_base(f, torch.float64)
    _, _, k = _solve(spl, P0d, f.t_r, [10.0 * i for i in range(8)], "1", monkeypatch)   # fp64 by default
    assert k == "fp64"
    g = Flux(f.t_r, 3000, f.tau, f.sigma, f.signal, f.background)               # N % 128 != 0
    P0r = spl.build_base(g, torch.float32)
    _, _, k = _solve(spl, P0r, g.t_r, [10.0 * i for i in range(8)], "1", monkeypatch)
    assert k == "fp64"


def test_i8_largest_n(spl, monkeypatch):
    """N = 66048, the largest N the int8 kernels take (u8 x u8 sums over N rows < 2^32), on a nearly
    flat flux: the encoded building plan, the converter kernel on the IEEE matrix and the FP64 GEMV
    agree."""
    N = 66048
    f = Flux(100.0, N, (50.0,), (1.0,), (1e-4,), 0.1)
    T = np.array([[10.0, 30.0, 50.0, 70.0, 90.0, 110.0, 130.0, 150.0]])
    monkeypatch.setenv("SPLIDAR_FUSED", "0")
    P0 = spl.empty_matrix(N, torch.float32, n_matrices=1)
    pe = spl.Plan(P0, f.t_r, T, tol=1e-12, build=[f])
    ie = pe.execute()
    assert pe.gemv() == "tensor_i8" and pe.storage() == "encoded"
    pie = pe.pi.detach().cpu().numpy().copy()
    pe.close()
    spl.build_base(f, torch.float32, out=P0[0])
    pic, ic, kc = _solve(spl, P0[0], f.t_r, T, "1", monkeypatch)
    pif, iff, kf = _solve(spl, P0[0], f.t_r, T, "0", monkeypatch)
    assert kc == "tensor_i8" and kf == "fp64"
    assert [i["iters"] for i in ie] == [i["iters"] for i in ic]
    assert all(abs(a["iters"] - b["iters"]) <= 1 for a, b in zip(ic, iff))
    assert np.max(np.sum(np.abs(pie - pic), axis=-1)) <= 1e-14
    assert np.max(np.sum(np.abs(pic - pif), axis=-1)) <= 1e-12


def test_i8_accumulator_beyond_2_31(spl, monkeypatch):
    """A constant matrix c = 1.99 2^-17 at N = 66048 from the uniform start: the top byte of every
    scaled entry (sig << 8) is 254 and so is the top byte of every x slice (1/N = 0.992 2^-16), so the
    most significant plane-times-slice sum is 254^2 N = 4.26e9: above 2^31 (where a signed read of the
    s32 accumulator goes wrong), below 2^32. y = c sum(x) for every column: pi stays uniform."""
    N = 66048
    c = np.float32(1.99 * 2.0 ** -17)
    assert ((int(np.array([c]).view(np.uint32)[0]) & 0x7FFFFF | 0x800000) >> 16) == 254
    P0 = spl.empty_matrix(N, torch.float32)
    P0.fill_(float(c))
    monkeypatch.setenv("SPLIDAR_I8", "1")
    plan = spl.Plan(P0, 100.0, np.array([[10.0, 30.0, 50.0, 70.0, 90.0, 110.0, 130.0, 150.0]]), tol=1e-12,
                    max_iter=20)                # a wrong product fails fast instead of iterating on
    i8 = plan.execute(check=False)
    assert plan.gemv() == "tensor_i8"
    pi8 = plan.pi.detach().cpu().numpy().copy()
    plan.close()
    assert all(i["converged"] for i in i8)
    assert np.max(np.abs(pi8 - 1.0 / N)) <= 1e-18
