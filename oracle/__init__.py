"""ORACLE — TEST INFRASTRUCTURE ONLY (see oracle/oracle.c header).

ctypes access to liboracle.so, the plain fp64 CPU implementation of arXiv 2509.20500 written from
PAPER.md. Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg
may import this module. It never imports the product package and the product never imports it.

Functions (each follows the passage cited in oracle.c):
  lam(flux, t), F(flux, t), Lambda(flux)     Eq. 1, S/B/Lambda, F (Thm 1)
  build_eq4(flux, t_d) -> P~ [N, N]          Eq. 3 bounds, D, Eq. 4, rows /sum
  rows_eq4(flux, t_d, r0, r1)                rows [r0, r1) of the same
  entry_eq4_unnorm(flux, t_d, i, j)          one unnormalised Eq. 4 entry
  left_matvec_streamed(flux, t_d, x)         x^T P~ with P~ recomputed row by row (large N)
  left_matvec_streamed_multi(flux, t_d, X)   the same for the rows of X, each P~ row computed once
  stationary_dense(P~), stationary_power(P~) pi P~ = pi
  monte_carlo(flux, t_d, ...)                continuous-time detection process of P:60
  second_eigenvalue(P), mixing_steps(P, pi), bin_trajectory(P, start, bin, steps)   §4
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")


def build(force: bool = False) -> str:
    """Compile oracle.c with gcc (IEEE fp64, no fast-math; OpenMP over rows only)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-std=c11",
                               "-fno-fast-math", "-ffp-contract=off", "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


class _Flux(C.Structure):
    _fields_ = [("t_r", C.c_double), ("n_bins", C.c_int32), ("n_pulses", C.c_int32),
                ("tau", C.POINTER(C.c_double)), ("sigma", C.POINTER(C.c_double)),
                ("signal", C.POINTER(C.c_double)), ("background", C.c_double)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(build())
        d, i32, i64, p = C.c_double, C.c_int32, C.c_int64, C.c_void_p
        fp = C.POINTER(_Flux)
        sig = {
            "oracle_lambda": (d, [fp, d]), "oracle_F": (d, [fp, d]), "oracle_Lambda": (d, [fp]),
            "oracle_Ftilde": (d, [fp, i64, d]),
            "oracle_entry_eq4_unnorm": (d, [fp, d, i32, i32]),
            "oracle_row_eq4": (C.c_int, [fp, d, i32, p]),
            "oracle_rows_eq4": (C.c_int, [fp, d, i32, i32, p]),
            "oracle_build_eq4": (C.c_int, [fp, d, p]),
            "oracle_left_matvec_streamed": (C.c_int, [fp, d, p, p]),
            "oracle_left_matvec_streamed_multi": (C.c_int, [fp, d, i32, p, p]),
            "oracle_stationary_dense": (C.c_int, [i32, p, p]),
            "oracle_stationary_power": (C.c_int, [i32, p, d, i32, p, C.POINTER(i32), C.POINTER(d)]),
            "oracle_mc": (C.c_int, [fp, d, C.c_uint64, i64, i64, i32, i32, p]),
            "oracle_mc_timestamps": (C.c_int, [fp, d, C.c_uint64, i64, p, p]),
            "oracle_left_matvec": (None, [i32, i32, p, p, p]),
            "oracle_set_threads": (None, [i32]),
            "oracle_max_threads": (i32, []),
        }
        for name, (res, args) in sig.items():
            fn = getattr(_lib, name)
            fn.restype, fn.argtypes = res, args
    return _lib


class _FluxRef:
    """Keeps the ctypes struct and the arrays it points to alive together."""

    def __init__(self, flux):
        self.tau = np.ascontiguousarray(flux.tau, dtype=np.float64)
        self.sigma = np.ascontiguousarray(flux.sigma, dtype=np.float64)
        self.signal = np.ascontiguousarray(flux.signal, dtype=np.float64)
        dp = C.POINTER(C.c_double)
        self.s = _Flux(float(flux.t_r), int(flux.n_bins), len(self.tau),
                       self.tau.ctypes.data_as(dp), self.sigma.ctypes.data_as(dp),
                       self.signal.ctypes.data_as(dp), float(flux.background))

    @property
    def ref(self):
        return C.byref(self.s)


def lam(flux, t: float) -> float:
    r = _FluxRef(flux)
    return lib().oracle_lambda(r.ref, float(t))


def F(flux, t: float) -> float:
    r = _FluxRef(flux)
    return lib().oracle_F(r.ref, float(t))


def Lambda(flux) -> float:
    r = _FluxRef(flux)
    return lib().oracle_Lambda(r.ref)


def Ftilde(flux, q: int, t: float) -> float:
    r = _FluxRef(flux)
    return lib().oracle_Ftilde(r.ref, int(q), float(t))


def entry_eq4_unnorm(flux, t_d: float, i: int, j: int) -> float:
    r = _FluxRef(flux)
    return lib().oracle_entry_eq4_unnorm(r.ref, float(t_d), int(i), int(j))


def rows_eq4(flux, t_d: float, r0: int, r1: int) -> np.ndarray:
    n = flux.n_bins
    out = np.empty((r1 - r0, n), dtype=np.float64)
    r = _FluxRef(flux)
    if lib().oracle_rows_eq4(r.ref, float(t_d), int(r0), int(r1), out.ctypes.data):
        raise ArithmeticError("oracle: zero or non-finite row sum")
    return out


def build_eq4(flux, t_d: float) -> np.ndarray:
    return rows_eq4(flux, t_d, 0, flux.n_bins)


def left_matvec_streamed_multi(flux, t_d: float, X: np.ndarray) -> np.ndarray:
    """Y[v] = X[v]^T P~ for the rows X[v] of X [k, N], every Eq. 4 row computed once."""
    X = np.ascontiguousarray(np.atleast_2d(X), dtype=np.float64)
    assert X.shape[1] == flux.n_bins
    Y = np.empty_like(X)
    r = _FluxRef(flux)
    if lib().oracle_left_matvec_streamed_multi(r.ref, float(t_d), int(X.shape[0]), X.ctypes.data, Y.ctypes.data):
        raise ArithmeticError("oracle: streamed matvec failed")
    return Y


def left_matvec_streamed(flux, t_d: float, x: np.ndarray) -> np.ndarray:
    x = np.ascontiguousarray(x, dtype=np.float64)
    y = np.empty(flux.n_bins, dtype=np.float64)
    r = _FluxRef(flux)
    if lib().oracle_left_matvec_streamed(r.ref, float(t_d), x.ctypes.data, y.ctypes.data):
        raise ArithmeticError("oracle: streamed matvec failed")
    return y


def left_matvec(rows: np.ndarray, x: np.ndarray) -> np.ndarray:
    """y = x^T rows (long double accumulation), the product inside stationary_power."""
    rows = np.ascontiguousarray(rows, dtype=np.float64)
    x = np.ascontiguousarray(x, dtype=np.float64)
    y = np.empty(rows.shape[1], dtype=np.longdouble)
    lib().oracle_left_matvec(rows.shape[0], rows.shape[1], rows.ctypes.data, x.ctypes.data, y.ctypes.data)
    return y.astype(np.float64)


def stationary_dense(P: np.ndarray) -> np.ndarray:
    P = np.ascontiguousarray(P, dtype=np.float64)
    n = P.shape[0]
    pi = np.empty(n, dtype=np.float64)
    if lib().oracle_stationary_dense(n, P.ctypes.data, pi.ctypes.data):
        raise ArithmeticError("oracle: singular system")
    return pi


def stationary_power(P: np.ndarray, tol: float = 1e-14, max_iter: int = 100000):
    """Returns (pi, iters, last L1 change, converged)."""
    P = np.ascontiguousarray(P, dtype=np.float64)
    n = P.shape[0]
    pi = np.empty(n, dtype=np.float64)
    it, ch = C.c_int32(0), C.c_double(0.0)
    st = lib().oracle_stationary_power(n, P.ctypes.data, float(tol), int(max_iter), pi.ctypes.data,
                                       C.byref(it), C.byref(ch))
    if st == 2:
        raise MemoryError("oracle: allocation failed")
    return pi, it.value, ch.value, st == 0


def monte_carlo(flux, t_d: float, seed: int, n_burn: int, n_per_batch: int, n_batches: int,
                n_hist: int) -> np.ndarray:
    """Histogram counts [n_batches, n_hist] of registered timestamps."""
    h = np.zeros((n_batches, n_hist), dtype=np.int64)
    r = _FluxRef(flux)
    if lib().oracle_mc(r.ref, float(t_d), int(seed), int(n_burn), int(n_per_batch), int(n_batches),
                       int(n_hist), h.ctypes.data):
        raise ValueError("oracle_mc: zero total flux")
    return h


def mc_timestamps(flux, t_d: float, seed: int, n: int):
    """The first n registrations (period q, offset t = T mod t_r) of one detection chain whose
    splitmix64 generator starts at `seed` (time starts at q = 0, t = 0)."""
    q = np.zeros(n, dtype=np.int64)
    t = np.zeros(n, dtype=np.float64)
    r = _FluxRef(flux)
    if lib().oracle_mc_timestamps(r.ref, float(t_d), int(seed) & (2 ** 64 - 1), int(n), q.ctypes.data, t.ctypes.data):
        raise ValueError("oracle_mc_timestamps: zero total flux")
    return q, t


def set_threads(n: int) -> None:
    """OpenMP threads of the row loops (timing only)."""
    lib().oracle_set_threads(int(n))


def max_threads() -> int:
    return int(lib().oracle_max_threads())


def shift_l(flux, t_d: float) -> int:
    """l = ceil(x_d / Delta) mod N (Thm 2) with x_d / Delta read as
    fmod(t_d, t_r) * N / t_r (reading R4). Used by oracle-side pins only."""
    import math
    u = math.fmod(float(t_d), flux.t_r) * flux.n_bins / flux.t_r
    if abs(u - round(u)) <= 8.0 * 2.220446049250313e-16 * max(1.0, abs(u)):
        u = float(round(u))                      # whole bins in decimal land on a bin centre (R4)
    return int(math.ceil(u)) % flux.n_bins


# ------------------------------------------------------------------ spectral analysis (§4)
# Plain definitions on a dense transition matrix (the oracle's Eq. 4 P~, or any row-stochastic
# matrix); numpy.linalg.eigvals and matmul are the library steps. SURVEY §8(f) row f1.

def second_eigenvalue(P: np.ndarray) -> complex:
    """lambda_2 of P (§4: "the magnitude of the second largest eigenvalue |lambda_2| of P~"):
    all eigenvalues by numpy.linalg.eigvals, drop the Perron root (the one closest to 1), return the
    largest-modulus remaining one; of a conjugate pair the member with phase in [0, pi]."""
    ev = np.linalg.eigvals(np.asarray(P, dtype=np.float64))
    k = int(np.argmin(np.abs(ev - 1.0)))
    rest = np.delete(ev, k)
    if rest.size == 0:
        return 0j
    mod = np.abs(rest)
    top = rest[np.abs(mod - mod.max()) <= 1e-12 * max(1.0, mod.max())]
    lam = top[np.argmax(top.imag)]                      # conjugate pair -> im >= 0
    return complex(lam.real, abs(lam.imag)) if abs(lam.imag) > 0 else complex(lam.real, 0.0)


def mixing_steps(P: np.ndarray, pi: np.ndarray, eps: float = 1e-3, max_steps: int = 100000):
    """§4.1: the smallest n >= 1 with max_i 1/2 ||e_i^T P^n - pi||_1 <= eps, by repeated
    multiplication of the full matrix power (every row is one start e_i). Returns (n, per-start first
    hits n_i) with n = -1 if max_steps is exceeded."""
    P = np.asarray(P, dtype=np.float64)
    pi = np.asarray(pi, dtype=np.float64)
    n_rows = P.shape[0]
    first = np.full(n_rows, -1, dtype=np.int64)
    Pn = P.copy()
    n_mix = -1
    for n in range(1, max_steps + 1):
        tv = 0.5 * np.abs(Pn - pi[None, :]).sum(axis=1)
        first[(first < 0) & (tv <= eps)] = n
        if n_mix < 0 and tv.max() <= eps:
            n_mix = n
        if np.all(first >= 0):
            break
        Pn = Pn @ P
    return n_mix, first


def bin_trajectory(P: np.ndarray, start: np.ndarray, bin: int, steps: int):
    """§4.2: (start^T P^n)[bin] for n = 0..steps, and start^T P^steps."""
    v = np.asarray(start, dtype=np.float64).copy()
    P = np.asarray(P, dtype=np.float64)
    out = [v[bin]]
    for _ in range(steps):
        v = v @ P
        out.append(v[bin])
    return np.array(out), v
