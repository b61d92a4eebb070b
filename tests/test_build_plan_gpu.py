"""Building plans (splidar_plan_create_build): every launch builds P~0 and solves, the first product
taken from the build's column sums (x^0 = 1/N: (1/N) 1^T J_l P~0 = (1/N) 1^T P~0, the row
permutation leaves column sums unchanged -- Thm 2). Against the separate build + plan:
the same iteration counts and pi to rounding, on every GEMV kind (fused, FP64, int8), in graph and
eager mode, for several matrices, and after new parameters (set_fluxes); against the oracle's Eq. 4
residual."""
import numpy as np
import pytest
import torch

import oracle
from workloads import Flux, config, random_flux

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def spl():
    assert torch.cuda.is_available(), "GPU tests need a B200"
    from paper_2509_20500_b200 import build
    build.build()
    import paper_2509_20500_b200 as s
    return s


def _pair(spl, fl, T, dtype, mode="factored"):
    N = fl[0].n_bins
    P0 = spl.empty_matrix(N, dtype, n_matrices=len(fl))
    pa = spl.Plan(P0, fl[0].t_r, T, tol=1e-12, build=fl, mode=mode)
    ia = pa.execute()
    pia = pa.pi.detach().cpu().numpy().copy()
    kind = pa.gemv()
    spl.build_base_batched(fl, dtype, mode, out=P0)
    pb = spl.Plan(P0, fl[0].t_r, T, tol=1e-12)
    ib = pb.execute()
    pib = pb.pi.detach().cpu().numpy().copy()
    pa.close()
    pb.close()
    return pia, ia, pib, ib, kind


def _c5(N):
    f0 = config(5).items[0].flux
    return Flux(f0.t_r, N, f0.tau, f0.sigma, f0.signal, f0.background)


@pytest.mark.parametrize("N,V,dtype,eager", [(256, 1, torch.float64, "0"), (4096, 17, torch.float64, "0"),
                                             (4096, 17, torch.float32, "0"), (4096, 17, torch.float32, "1"),
                                             (5000, 2, torch.float64, "1"), (9001, 1, torch.float32, "0")])
def test_building_plan_equals_separate(spl, monkeypatch, N, V, dtype, eager):
    monkeypatch.setenv("SPLIDAR_EAGER", eager)
    f = _c5(N)
    w = config(5)
    T = np.array([([w.items[0].t_d] + [it.t_d for it in w.sweep])[:V]])
    pia, ia, pib, ib, kind = _pair(spl, [f], T, dtype)
    assert [i["iters"] for i in ia] == [i["iters"] for i in ib]
    assert all(i["converged"] for i in ia)
    assert np.max(np.sum(np.abs(pia - pib), axis=-1)) <= 1e-14
    if dtype == torch.float32 and V >= 8:
        assert kind == "tensor_i8"
    y = oracle.left_matvec_streamed(f, T[0, 0], pia[0, 0])
    assert np.sum(np.abs(y - pia[0, 0])) <= (1e-11 if dtype == torch.float64 else 1e-5)


def test_building_plan_batched_and_exp(spl):
    rng = np.random.default_rng(21)
    fl = [random_flux(rng, 4096, 1) for _ in range(5)]
    fl = [Flux(100.0, 4096, f.tau, f.sigma, f.signal, f.background) for f in fl]
    T = rng.uniform(0, 250, (5, 1))
    for mode in ("factored", "exp"):
        pia, ia, pib, ib, _ = _pair(spl, fl, T, torch.float64, mode)
        assert [i["iters"] for i in ia] == [i["iters"] for i in ib]
        assert np.max(np.sum(np.abs(pia - pib), axis=-1)) <= 1e-14


def test_set_fluxes(spl):
    """New theta through set_fluxes gives the plan built for that theta."""
    c4 = config(4).items[0]
    f = c4.flux
    g = Flux(f.t_r, f.n_bins, (60.0,), (0.2,), (1.5,), 0.7)
    P0 = spl.empty_matrix(f.n_bins, torch.float64)
    plan = spl.Plan(P0, f.t_r, [[c4.t_d]], tol=1e-12, build=[f])
    plan.execute()
    plan.set_fluxes([g])
    ig = plan.execute()
    got = plan.pi[0, 0].detach().cpu().numpy().copy()
    plan.close()
    P1 = spl.build_base(g, torch.float64)
    ref, ir = spl.stationary(P1, g.t_r, c4.t_d)
    assert ig[0]["iters"] == ir["iters"]
    assert np.sum(np.abs(got - ref.cpu().numpy())) <= 1e-14
    with pytest.raises(spl.SplidarError):
        plan2 = spl.Plan(P0, f.t_r, [[c4.t_d]], build=[f])
        plan2.set_fluxes([Flux(f.t_r, 1024, f.tau, f.sigma, f.signal, f.background)])   # other N


def test_building_plan_range_test(spl):
    """The int8 GEMV's column exponents and range test come from the build of a building plan: a
    flux whose columns span more than 2^8 (Lambda = 61) must run the FP64 GEMV, a moderate one the
    int8 GEMV, both equal to the separate build + plan."""
    tds = [[10.0, 30.0, 50.0, 70.0, 90.0, 110.0, 130.0, 150.0]]
    for sig, want in ((60.0, "fp64"), (1.0, "tensor_i8")):
        f = Flux(200.0, 4096, (60.0,), (0.5,), (sig,), 1.0)
        pia, ia, pib, ib, kind = _pair(spl, [f], np.array(tds), torch.float32)
        assert kind == want
        assert [i["iters"] for i in ia] == [i["iters"] for i in ib]
        assert np.max(np.sum(np.abs(pia - pib), axis=-1)) <= 1e-13


def test_building_plan_batched_int8(spl, monkeypatch):
    """M = 3 matrices x 8 dead times on the int8 GEMV, matrices and exponents built by the plan."""
    rng = np.random.default_rng(33)
    fl = [random_flux(rng, 2048, 2, sigma_bins=(1, 10), s_range=(0.5, 1.5), b_range=(0.2, 1.0)) for _ in range(3)]
    fl = [Flux(100.0, 2176, f.tau, f.sigma, f.signal, f.background) for f in fl]
    T = rng.uniform(0, 300, (3, 8))
    monkeypatch.setenv("SPLIDAR_FUSED", "0")
    pia, ia, pib, ib, kind = _pair(spl, fl, T, torch.float32)
    assert kind == "tensor_i8"
    assert [i["iters"] for i in ia] == [i["iters"] for i in ib]
    assert np.max(np.sum(np.abs(pia - pib), axis=-1)) <= 1e-13


def _encode_ref(P):
    """Test-side encoding of an fp32 matrix: column j's entries as sig << (e - E_j + 8), E_j the
    column's largest biased exponent (the int8 GEMV's scaled integers); None if out of range."""
    u = P.view(np.uint32).astype(np.uint64)
    e = ((u >> 23) & 0xFF).astype(np.int64)
    nz = (u & 0x7FFFFFFF) != 0
    E = np.where(nz, e, 0).max(axis=0)
    emin = np.where(nz, e, 1 << 20).min(axis=0)
    has = emin < (1 << 20)                          # columns with a non-zero entry (all-zero ones encode as 0)
    if np.any(has & (E - emin > 8)) or np.any(has & (E <= 8)) or np.any(nz & (e == 0)):
        return None
    sig = (u & 0x7FFFFF) | 0x800000
    sh = e - E[None, :] + 8
    w = np.where(nz, sig << np.clip(sh, 0, 63).astype(np.uint64), 0)
    assert np.all(w < 2 ** 32)
    return w.astype(np.uint32)


@pytest.mark.parametrize("enc_env", ["1", "0"])
def test_building_plan_encoded_storage(spl, monkeypatch, enc_env):
    """fp32 factored building plans on the int8 GEMV store P~0 encoded: every entry as its column's
    scaled integer, with the column exponents derived from 1/D before the build (k_enc_colexp). The
    stored words must equal the test-side encoding of the separately built fp32 matrix, bit for bit
    (SPLIDAR_I8_ENC=0: plain fp32), and pi must equal the separate plan's."""
    monkeypatch.setenv("SPLIDAR_I8_ENC", enc_env)
    rng = np.random.default_rng(5)
    w = config(5)
    for N, f in ((4096, _c5(4096)), (2176, random_flux(rng, 2176, 2, sigma_bins=(1, 10), s_range=(0.5, 1.5),
                                                       b_range=(0.2, 1.0)))):
        f = Flux(f.t_r, N, f.tau, f.sigma, f.signal, f.background)
        T = np.array([([w.items[0].t_d] + [it.t_d for it in w.sweep])[:17]])
        monkeypatch.setenv("SPLIDAR_FUSED", "0")
        P0 = spl.empty_matrix(N, torch.float32, n_matrices=1)
        pa = spl.Plan(P0, f.t_r, T, tol=1e-12, build=[f])
        ia = pa.execute()
        assert pa.gemv() == "tensor_i8"
        assert pa.storage() == ("encoded" if enc_env == "1" else "ieee")
        stored = P0[0].contiguous().cpu().numpy()
        pia = pa.pi.detach().cpu().numpy().copy()
        pa.close()
        ref = spl.build_base(f, torch.float32).cpu().numpy()
        want = _encode_ref(ref)
        assert want is not None
        if enc_env == "1":
            assert np.array_equal(stored.view(np.uint32), want)
        else:
            assert np.array_equal(stored.view(np.uint32), ref.view(np.uint32))
        pb = spl.Plan(spl.build_base(f, torch.float32), f.t_r, T, tol=1e-12)
        ib = pb.execute()
        pib = pb.pi.detach().cpu().numpy().copy()
        pb.close()
        assert [i["iters"] for i in ia] == [i["iters"] for i in ib]
        assert np.max(np.sum(np.abs(pia - pib), axis=-1)) <= 1e-13


@pytest.mark.parametrize("sig,bg,want_enc", [(60.0, 1.0, False), (5.0, 0.05, None), (5.5, 0.01, None), (1.0, 1.0, True)])
def test_building_plan_encoded_range(spl, sig, bg, want_enc):
    """The range test from 1/D (before the build) agrees with the range test of the stored fp32
    matrix: columns spanning more than 2^8 (Lambda = 61; Lambda ~ 5 sits near the edge, either way)
    fall back to plain fp32 storage and the FP64 GEMV (the stored matrix equals the separate fp32
    build, bit for bit); otherwise the words equal the test-side encoding."""
    f = Flux(200.0, 4096, (60.0,), (0.5,), (sig,), bg)
    T = np.array([[10.0, 30.0, 50.0, 70.0, 90.0, 110.0, 130.0, 150.0]])
    ref = spl.build_base(f, torch.float32).cpu().numpy()
    want = _encode_ref(ref)
    if want_enc is not None:
        assert (want is not None) == want_enc
    P0 = spl.empty_matrix(4096, torch.float32, n_matrices=1)
    pa = spl.Plan(P0, f.t_r, T, tol=1e-12, build=[f])
    pa.execute()
    stored = P0[0].contiguous().cpu().numpy().view(np.uint32)
    if want is None:
        assert pa.gemv() == "fp64" and pa.storage() == "ieee"
        assert np.array_equal(stored, ref.view(np.uint32))
    else:
        assert pa.gemv() == "tensor_i8" and pa.storage() == "encoded"
        assert np.array_equal(stored, want)
    pa.close()


@pytest.mark.parametrize("N,V,M", [(1152, 18, 1), (2176, 19, 1), (1024, 8, 4), (8192, 12, 2)])
def test_building_plan_fp32_shapes(spl, monkeypatch, N, V, M):
    """fp32 building plans at the edges of the int8 path: the most dead times it takes (18), one more
    (19: the FP64 kernel with 24 slots), the smallest N (1024) with several matrices, and 12 dead
    times on two larger matrices; each equal to the separate build + plan."""
    monkeypatch.setenv("SPLIDAR_FUSED", "0")
    rng = np.random.default_rng(N + V + M)
    fl = [random_flux(rng, N, 2, sigma_bins=(1, 10), s_range=(0.5, 1.5), b_range=(0.2, 1.0)) for _ in range(M)]
    fl = [Flux(100.0, N, f.tau, f.sigma, f.signal, f.background) for f in fl]
    T = rng.uniform(0, 300, (M, V))
    pia, ia, pib, ib, kind = _pair(spl, fl, T, torch.float32)
    assert kind == ("tensor_i8" if V <= 18 else "fp64")
    assert [i["iters"] for i in ia] == [i["iters"] for i in ib]
    assert all(i["converged"] for i in ia)
    assert np.max(np.sum(np.abs(pia - pib), axis=-1)) <= 1e-13


@pytest.mark.parametrize("N,dtype", [(256, torch.float64), (1024, torch.float64), (700, torch.float32)])
def test_fused_building_plan_graph_replay(spl, N, dtype):
    """Small-N building plans launch steps 1-4 as one cached graph on a stream that is not capturing,
    and as kernels into a caller's capture: both equal the separate build + plan, across replays and
    after set_fluxes (the graph reads theta from the workspace, so it is not re-captured)."""
    f = _c5(N)
    g = Flux(f.t_r, N, (37.0, 120.0), (0.3, 0.2), (1.2, 0.4), 0.3)
    T = np.array([[55.0, 430.0]])
    P0 = spl.empty_matrix(N, dtype)
    plan = spl.Plan(P0, f.t_r, T, tol=1e-12, build=[f])
    assert plan.fused
    for flux in (f, g, f):
        plan.set_fluxes([flux])
        i1 = plan.execute()
        p1 = plan.pi.clone()
        i2 = plan.execute()                                   # replay
        assert i1 == i2 and torch.equal(p1, plan.pi)
        st = torch.cuda.Stream()
        graph = torch.cuda.CUDAGraph()                        # the caller's capture: direct kernels
        with torch.cuda.graph(graph, stream=st):
            plan.launch(stream=st)
        graph.replay()
        torch.cuda.synchronize()
        assert plan.info() == i1 and torch.equal(p1, plan.pi)
        P1 = spl.build_base(flux, dtype)
        ref = spl.Plan(P1, flux.t_r, T, tol=1e-12)
        ir = ref.execute()
        assert [i["iters"] for i in ir] == [i["iters"] for i in i1]
        assert torch.sum(torch.abs(ref.pi - plan.pi)).item() <= 1e-14
        ref.close()
    plan.close()
