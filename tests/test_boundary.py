"""The C-ABI boundary on the CPU: the library loads without a GPU, exports every symbol that
include/splidar.h declares, and its host-side logic (shift rule, workspace sizing, argument
validation, status strings) behaves as documented. No compute is launched here."""
import ctypes as C
import math
import os
import re

import numpy as np
import pytest

import oracle
from workloads import config, parity_cases

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "splidar.h")


@pytest.fixture(scope="module")
def spl():
    from paper_2509_20500_b200 import build
    build.build()
    import paper_2509_20500_b200.splidar as s
    s._lib()
    return s


def _declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    names = re.findall(r"\b(splidar_[a-z_]+)\s*\(", src)
    return sorted(set(names))


def test_header_declares_the_path():
    names = _declared_functions()
    for must in ("splidar_build_base", "splidar_apply_deadtime", "splidar_stationary", "splidar_sweep",
                 "splidar_flux_vectors", "splidar_shift", "splidar_workspace_bytes"):
        assert must in names


def test_library_exports_every_declared_symbol(spl):
    lib = C.CDLL(spl.LIB_PATH)
    missing = [n for n in _declared_functions() if not hasattr(lib, n)]
    assert not missing, missing


def test_build_info(spl):
    assert "sm_100a" in spl.build_info()


def test_status_strings(spl):
    for st in range(6):
        assert spl._lib().splidar_strerror(st).decode()
    assert spl._lib().splidar_strerror(99).decode() == "unknown status"


# ------------------------------------------------------------------ shift rule (Thm 2)
def test_shift_rule_config_values(spl):
    """l = ceil(x_d / Delta) mod N at the BASELINE configs."""
    want = {1: 192, 2: 512, 3: 3277, 4: 3277, 5: 4916}
    for k, l in want.items():
        w = config(k)
        f = w.items[0].flux
        assert spl.shift(f.t_r, f.n_bins, w.items[0].t_d) == l
    w = config(5)
    f = w.items[0].flux
    got = [spl.shift(f.t_r, f.n_bins, it.t_d) for it in w.sweep]
    assert got == [1639, 6991, 12343, 17695, 23047, 28399, 984, 6336, 11688, 17040, 22392, 27744,
                   328, 5680, 11032, 16384]


def test_shift_rule_matches_oracle_and_edges(spl):
    rng = np.random.default_rng(4)
    for _ in range(500):
        n = int(rng.integers(2, 70000))
        t_r = float(rng.uniform(1, 300))
        td = float(rng.uniform(0, 4 * t_r))
        assert spl.shift(t_r, n, td) == oracle.shift_l(_F(t_r, n), td)
    assert spl.shift(100.0, 256, 0.0) == 0
    assert spl.shift(100.0, 256, 100.0) == 0           # whole period
    assert spl.shift(100.0, 256, 300.0) == 0
    assert spl.shift(100.0, 4, 99.0) == 0               # l = N wraps to 0
    assert spl.shift(100.0, 4, 25.0) == 1               # exact integer: ceil(1) = 1
    assert spl.shift(100.0, 4, 25.0001) == 2
    # whole bins written in decimal (Delta = 0.1, 0.01 not binary fractions): the re-arm point lands
    # on a bin centre (reading R4), never one bin further; l = N wraps to 0
    assert spl.shift(1.0, 10, 0.3) == 3                 # 0.3 * 10 / 1 = 3.0000000000000004 in fp64
    assert spl.shift(0.1, 10, 0.3) == 0                 # fmod(0.3, 0.1) = 0.0999..: u ~ N -> l = 0
    for k in (1, 3, 7, 29, 113, 4321):
        td = float(f"{k / 100:.2f}")                    # k Delta, Delta = 0.01 (t_r = 100, N = 10000)
        assert spl.shift(100.0, 10000, td) == k == oracle.shift_l(_F(100.0, 10000), td)


class _F:
    def __init__(self, t_r, n):
        self.t_r, self.n_bins = t_r, n


@pytest.mark.parametrize("args", [(0.0, 16, 1.0), (-1.0, 16, 1.0), (100.0, 1, 1.0), (100.0, 16, -1.0),
                                  (math.inf, 16, 1.0), (100.0, 16, math.nan)])
def test_shift_rejects(spl, args):
    out = C.c_int32(0)
    assert spl._lib().splidar_shift(*args, C.byref(out)) == spl.EINVAL


# ------------------------------------------------------------------ workspace sizing
def test_workspace_bytes(spl):
    assert spl.workspace_bytes(1, 1, 1) == 0
    assert spl.workspace_bytes(256, 0, 1) == 0
    assert spl.workspace_bytes(256, 1, 33) == 0
    a = spl.workspace_bytes(32768, 1, 1)
    b = spl.workspace_bytes(32768, 1, 32)
    assert 0 < a < b
    assert b < 1 << 30                     # < 1 GiB beside an 8.6 GB matrix
    assert spl.workspace_bytes(4096, 64, 1) > spl.workspace_bytes(4096, 1, 1)
    for n in (2, 3, 255, 1537, 32768):
        assert spl.workspace_bytes(n, 1, 1) % 256 == 0


# ------------------------------------------------------------------ argument validation (no launch)
def _flux_struct(spl, **kw):
    f = config(1).items[0].flux
    d = dict(t_r=f.t_r, n_bins=f.n_bins, tau=f.tau, sigma=f.sigma, signal=f.signal, background=f.background)
    d.update(kw)

    class Obj:
        pass
    o = Obj()
    for k, v in d.items():
        setattr(o, k, v)
    return spl._FluxArg(o)


FAKE = 1 << 20          # 256-aligned fake device address: validation must fail before any access


@pytest.mark.parametrize("kw", [dict(t_r=0.0), dict(n_bins=1), dict(n_bins=(1 << 20) + 1), dict(sigma=(0.0,)),
                                dict(signal=(-1.0,)), dict(tau=(100.0,)), dict(tau=(-0.1,)),
                                dict(background=0.0), dict(background=math.nan), dict(signal=(700.0,)),
                                dict(tau=tuple([1.0] * 17), sigma=tuple([1.0] * 17), signal=tuple([0.1] * 17))])
def test_build_base_rejects_bad_flux(spl, kw):
    fa = _flux_struct(spl, **kw)
    st = spl._lib().splidar_build_base(C.byref(fa.s), spl.F64, 0, FAKE, 256, FAKE, 1 << 30, None)
    assert st == spl.EINVAL


def test_build_base_rejects_layout(spl):
    fa = _flux_struct(spl)
    lib = spl._lib()
    assert lib.splidar_build_base(C.byref(fa.s), spl.F64, 0, FAKE, 255, FAKE, 1 << 30, None) == spl.ENOSPACE
    assert lib.splidar_build_base(C.byref(fa.s), spl.F64, 0, FAKE + 8, 256, FAKE, 1 << 30, None) == spl.ENOSPACE
    assert lib.splidar_build_base(C.byref(fa.s), spl.F32, 0, FAKE, 258, FAKE, 1 << 30, None) == spl.ENOSPACE
    assert lib.splidar_build_base(C.byref(fa.s), spl.F64, 0, FAKE, 256, FAKE, 16, None) == spl.ENOSPACE
    assert lib.splidar_build_base(C.byref(fa.s), spl.F64, 0, FAKE, 256, FAKE + 64, 1 << 30, None) == spl.ENOSPACE
    assert lib.splidar_build_base(C.byref(fa.s), spl.F64, 7, FAKE, 256, FAKE, 1 << 30, None) == spl.EINVAL
    assert lib.splidar_build_base(C.byref(fa.s), 3, 0, FAKE, 256, FAKE, 1 << 30, None) == spl.EINVAL
    assert lib.splidar_build_base(C.byref(fa.s), spl.F64, 0, None, 256, FAKE, 1 << 30, None) == spl.EINVAL


def test_apply_deadtime_rejects(spl):
    lib = spl._lib()
    assert lib.splidar_apply_deadtime(FAKE, FAKE, 256, 256, spl.F64, 100.0, 75.0, None) == spl.EINVAL
    assert lib.splidar_apply_deadtime(FAKE, FAKE * 2, 256, 256, spl.F64, 100.0, -1.0, None) == spl.EINVAL
    assert lib.splidar_apply_deadtime(FAKE, FAKE * 2, 256, 250, spl.F64, 100.0, 1.0, None) == spl.ENOSPACE


def test_stationary_rejects(spl):
    lib = spl._lib()
    info = spl.SolveInfo()
    ws = spl.workspace_bytes(256, 1, 1)
    args = dict(P0=FAKE, n=256, ld=256, dt=spl.F64, t_r=100.0, t_d=75.0, tol=1e-12, it=100, pi=FAKE, ws=FAKE,
                wsb=ws)

    def call(**kw):
        a = dict(args)
        a.update(kw)
        return lib.splidar_stationary(a["P0"], a["n"], a["ld"], a["dt"], a["t_r"], a["t_d"], a["tol"], a["it"],
                                      a["pi"], a["ws"], a["wsb"], C.byref(info), None)
    assert call(tol=0.0) == spl.EINVAL
    assert call(tol=math.nan) == spl.EINVAL
    assert call(it=0) == spl.EINVAL
    assert call(pi=None) == spl.EINVAL
    assert call(t_d=-5.0) == spl.EINVAL
    assert call(wsb=ws - 1) == spl.ENOSPACE
    assert call(ld=100) == spl.ENOSPACE


def test_second_eigenvalue_dense_rejects(spl):
    lib = spl._lib()
    info = spl.SpectralInfo()
    wsb = lib.splidar_spectral_dense_workspace_bytes(256)
    assert wsb >= spl.workspace_bytes(256, 1, 2) and lib.splidar_spectral_dense_workspace_bytes(1) == 0
    args = dict(P0=FAKE, n=256, ld=256, dt=spl.F64, t_r=100.0, t_d=75.0, pi=FAKE, tol=1e-13, it=100, ws=FAKE,
                wsb=wsb)

    def call(**kw):
        a = dict(args)
        a.update(kw)
        return lib.splidar_second_eigenvalue_dense(a["P0"], a["n"], a["ld"], a["dt"], a["t_r"], a["t_d"], a["pi"],
                                                   a["tol"], a["it"], a["ws"], a["wsb"], C.byref(info), None)
    assert call(n=1) == spl.EINVAL
    assert call(pi=None) == spl.EINVAL
    assert call(P0=None) == spl.EINVAL
    assert call(dt=7) == spl.EINVAL
    assert call(tol=0.0) == spl.EINVAL
    assert call(tol=math.inf) == spl.EINVAL
    assert call(it=1) == spl.EINVAL
    assert call(t_d=-1.0) == spl.EINVAL
    assert call(t_r=0.0) == spl.EINVAL
    assert call(ld=255) == spl.ENOSPACE
    assert call(wsb=wsb - 1) == spl.ENOSPACE
    assert call(ws=FAKE + 8) == spl.ENOSPACE


def test_sweep_rejects(spl):
    lib = spl._lib()
    fa = _flux_struct(spl)
    S = np.array([0.5, 1.0])
    B = np.array([0.1, 0.0])          # B = 0 is invalid (irreducibility)
    T = np.array([75.0, 75.0])
    st = lib.splidar_sweep(C.byref(fa.s), 2, S.ctypes.data, B.ctypes.data, T.ctypes.data, spl.F64, 0, 1e-12, 100,
                           FAKE, FAKE, 2, 256, FAKE, 1 << 30, None, None)
    assert st == spl.EINVAL
    B = np.array([0.1, 0.2])
    st = lib.splidar_sweep(C.byref(fa.s), 0, S.ctypes.data, B.ctypes.data, T.ctypes.data, spl.F64, 0, 1e-12, 100,
                           FAKE, FAKE, 2, 256, FAKE, 1 << 30, None, None)
    assert st == spl.EINVAL
    # P0_store = NULL: matrix-free (structured) path, validated as splidar_stationary_structured
    need = lib.splidar_structured_workspace_bytes(256, 2, 2)
    st = lib.splidar_sweep(C.byref(fa.s), 2, S.ctypes.data, B.ctypes.data, T.ctypes.data, spl.F64, 0, 1e-12, 100,
                           FAKE, None, 0, 0, FAKE, need - 1, None, None)
    assert st == spl.ENOSPACE
    B0 = np.array([0.1, 0.0])
    st = lib.splidar_sweep(C.byref(fa.s), 2, S.ctypes.data, B0.ctypes.data, T.ctypes.data, spl.F64, 0, 1e-12, 100,
                           FAKE, None, 0, 0, FAKE, need, None, None)
    assert st == spl.EINVAL


def test_parity_cases_are_well_formed():
    """The seeded parity workload spans tiny N, ragged tails (N not a multiple of the 512-column
    strip), several strips, K = 1 and 2 pulses, zero / whole-period / multi-period dead times."""
    cases = parity_cases()
    ns = {c.flux.n_bins for c in cases}
    assert {2, 3, 1000, 1537, 2048} <= ns
    assert any(c.t_d == 0.0 for c in cases) and any(c.t_d > 2 * c.flux.t_r for c in cases)
    assert any(c.flux.n_pulses == 2 for c in cases)


# ------------------------------------------------------------------ §8(f) entry points: host validation
def _items(S=(0.5,), B=(0.1,), T=(75.0,)):
    return (np.ascontiguousarray(S, dtype=np.float64), np.ascontiguousarray(B, dtype=np.float64),
            np.ascontiguousarray(T, dtype=np.float64))


def test_structured_workspace_bytes(spl):
    lib = spl._lib()
    assert lib.splidar_structured_workspace_bytes(65536, 1, 1) > 0          # a cluster of 16 CTAs
    assert lib.splidar_structured_workspace_bytes(65537, 1, 1) == 0         # beyond 16 x 4096 bins
    assert lib.splidar_structured_workspace_bytes(1, 1, 1) == 0
    assert lib.splidar_structured_workspace_bytes(256, 0, 1) == 0
    a = lib.splidar_structured_workspace_bytes(4096, 3, 10)
    assert a % 256 == 0 and lib.splidar_structured_workspace_bytes(4096, 3, 20) > a
    assert lib.splidar_mc_workspace_bytes(2, 5) > 0 and lib.splidar_mc_workspace_bytes(0, 5) == 0


def test_structured_rejects(spl):
    lib = spl._lib()
    fa = _flux_struct(spl)
    S, B, T = _items()
    ws = lib.splidar_structured_workspace_bytes(256, 1, 1)

    def solve(S=S, B=B, T=T, tol=1e-12, it=100, pi=FAKE, wsb=ws, n=1):
        return lib.splidar_stationary_structured(C.byref(fa.s), n, S.ctypes.data, B.ctypes.data, T.ctypes.data, tol,
                                                 it, pi, FAKE, wsb, None, None)
    assert solve(tol=0.0) == spl.EINVAL
    assert solve(it=0) == spl.EINVAL
    assert solve(pi=None) == spl.EINVAL
    assert solve(n=0) == spl.EINVAL
    assert solve(T=np.array([-1.0])) == spl.EINVAL
    assert solve(B=np.array([0.0])) == spl.EINVAL                           # B = 0: reducible chain (R16)
    assert solve(S=np.array([-0.5])) == spl.EINVAL
    assert solve(wsb=ws - 1) == spl.ENOSPACE
    info = spl.SpectralInfo()
    assert lib.splidar_second_eigenvalue(C.byref(fa.s), 1, S.ctypes.data, B.ctypes.data, T.ctypes.data, None, 1e-13,
                                         100, FAKE, ws, C.byref(info), None) == spl.EINVAL
    h = C.c_void_p(None)
    assert lib.splidar_splan_create(C.byref(h), 7, C.byref(fa.s), 1, S.ctypes.data, B.ctypes.data, T.ctypes.data,
                                    1e-12, 100, FAKE, FAKE, ws, None) == spl.EINVAL
    assert not h.value
    out = C.c_int32(0)
    wsm = lib.splidar_structured_workspace_bytes(256, 1, 256)
    assert lib.splidar_mixing_steps(C.byref(fa.s), 75.0, FAKE, 0.0, 100, None, C.byref(out), FAKE, wsm,
                                    None) == spl.EINVAL
    assert lib.splidar_mixing_steps(C.byref(fa.s), 75.0, FAKE, 1e-3, 100, None, C.byref(out), FAKE, wsm - 1,
                                    None) == spl.ENOSPACE
    assert lib.splidar_bin_trajectory(C.byref(fa.s), 75.0, FAKE, 256, 10, FAKE, None, FAKE, ws, None) == spl.EINVAL
    assert lib.splidar_bin_trajectory(C.byref(fa.s), 75.0, FAKE, 0, -1, FAKE, None, FAKE, ws, None) == spl.EINVAL


def test_monte_carlo_rejects(spl):
    lib = spl._lib()
    fa = _flux_struct(spl)
    S, B, T = _items()
    ws = lib.splidar_mc_workspace_bytes(1, 1)

    def mc(runs=4, split=1, burn=10, regs=100, cycles=0, nh=16, hist=FAKE, nrec=0, wsb=ws, T=T):
        return lib.splidar_monte_carlo(C.byref(fa.s), 1, S.ctypes.data, B.ctypes.data, T.ctypes.data, 1, runs, split,
                                       burn, regs, cycles, nh, hist, nrec, None, None, FAKE, wsb, None)
    assert mc(runs=0) == spl.EINVAL
    assert mc(split=0) == spl.EINVAL
    assert mc(regs=0, cycles=0) == spl.EINVAL
    assert mc(split=3, regs=100) == spl.EINVAL                              # budget not divisible by n_split
    assert mc(split=4, regs=0, cycles=50001) == spl.EINVAL
    assert mc(nh=0) == spl.EINVAL
    assert mc(hist=None) == spl.EINVAL
    assert mc(nrec=5) == spl.EINVAL                                         # records requested, no buffers
    assert mc(T=np.array([-2.0])) == spl.EINVAL
    assert mc(wsb=ws - 1) == spl.ENOSPACE


def test_build_eq4_rejects(spl):
    lib = spl._lib()
    fa = _flux_struct(spl)
    assert lib.splidar_build_eq4(C.byref(fa.s), -1.0, spl.F64, FAKE, 256, None) == spl.EINVAL
    assert lib.splidar_build_eq4(C.byref(fa.s), math.inf, spl.F64, FAKE, 256, None) == spl.EINVAL
    assert lib.splidar_build_eq4(C.byref(fa.s), 75.0, spl.F64, FAKE, 250, None) == spl.ENOSPACE
    assert lib.splidar_build_eq4(C.byref(fa.s), 75.0, spl.F64, None, 256, None) == spl.EINVAL
    bad = _flux_struct(spl, background=0.0)
    assert lib.splidar_build_eq4(C.byref(bad.s), 75.0, spl.F64, FAKE, 256, None) == spl.EINVAL


def test_plan_kind_null(spl):
    assert spl._lib().splidar_plan_kind(None) == -1
    assert spl._lib().splidar_plan_gemv(None, None) == -1
