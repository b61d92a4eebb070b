"""Thin Python binding of libsplidar.so (include/splidar.h): argument marshalling only.

Every step of the path runs in the library's sm_100a kernels; PyTorch supplies device memory,
streams and the current device. There is no CPU fallback: if the library is missing or fails to
load, every call raises.
"""
from __future__ import annotations

import contextlib
import ctypes as C
import functools
import inspect
import math
import os
from dataclasses import dataclass

import numpy as np
import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "lib", "libsplidar.so")

OK, EINVAL, ENOCONV, EZEROROW, ENOSPACE, ECUDA = range(6)
F64, F32 = 0, 1
ENTRY_FACTORED, ENTRY_EXP = 0, 1
MAX_PULSES = 16
MAX_VECTORS = 32

_DTYPES = {torch.float64: F64, torch.float32: F32}
_MODES = {"factored": ENTRY_FACTORED, "exp": ENTRY_EXP}


class SplidarError(RuntimeError):
    def __init__(self, status: int, where: str):
        self.status = status
        msg = _lib().splidar_strerror(status).decode()
        if status == ECUDA:
            msg += f" (cudaError {_lib().splidar_last_cuda_error()})"
        super().__init__(f"{where}: {msg} [status {status}]")


class _Flux(C.Structure):
    _fields_ = [("t_r", C.c_double), ("n_bins", C.c_int32), ("n_pulses", C.c_int32),
                ("tau", C.POINTER(C.c_double)), ("sigma", C.POINTER(C.c_double)),
                ("signal", C.POINTER(C.c_double)), ("background", C.c_double)]


class SolveInfo(C.Structure):
    _fields_ = [("iters", C.c_int32), ("converged", C.c_int32), ("shift_l", C.c_int32),
                ("reserved", C.c_int32), ("l1_change", C.c_double), ("lambda_total", C.c_double)]

    def as_dict(self) -> dict:
        return {"iters": self.iters, "converged": bool(self.converged), "shift_l": self.shift_l,
                "l1_change": self.l1_change, "lambda_total": self.lambda_total}


class SpectralInfo(C.Structure):
    _fields_ = [("lambda2_re", C.c_double), ("lambda2_im", C.c_double), ("modulus", C.c_double),
                ("phase", C.c_double), ("gap", C.c_double), ("change", C.c_double), ("iters", C.c_int32),
                ("converged", C.c_int32)]

    def as_dict(self) -> dict:
        return {"lambda2": complex(self.lambda2_re, self.lambda2_im), "modulus": self.modulus,
                "phase": self.phase, "gap": self.gap, "change": self.change, "iters": self.iters,
                "converged": bool(self.converged)}


_LIB = None


def _lib():
    global _LIB
    if _LIB is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"libsplidar.so not built ({LIB_PATH}); run "
                               "`python -m paper_2509_20500_b200.build` (no CPU fallback exists)")
        lib = C.CDLL(LIB_PATH)
        st, i32, i64, d, p, sz = C.c_int, C.c_int32, C.c_int64, C.c_double, C.c_void_p, C.c_size_t
        fp = C.POINTER(_Flux)
        pinfo = C.POINTER(SolveInfo)
        sig = {
            "splidar_shift": (st, [d, i32, d, C.POINTER(i32)]),
            "splidar_workspace_bytes": (sz, [i32, i32, i32]),
            "splidar_flux_vectors": (st, [fp, p, p, p, p, p, p, sz, p]),
            "splidar_build_base": (st, [fp, st, st, p, i64, p, sz, p]),
            "splidar_build_base_batched": (st, [fp, i32, st, st, p, i64, i64, p, sz, p]),
            "splidar_apply_deadtime": (st, [p, p, i32, i64, st, d, d, p]),
            "splidar_stationary": (st, [p, i32, i64, st, d, d, d, i32, p, p, sz, pinfo, p]),
            "splidar_stationary_multi": (st, [p, i32, i64, i32, i64, st, d, p, i32, d, i32, p, p, sz, pinfo, p]),
            "splidar_stationary_multi_host": (st, [p, i32, i64, i32, i64, st, d, p, i32, d, i32, p, p, p, sz, pinfo,
                                                   p]),
            "splidar_plan_cache_clear": (None, []),
            "splidar_sweep": (st, [fp, i32, p, p, p, st, st, d, i32, p, p, i32, i64, p, sz, pinfo, p]),
            "splidar_plan_create": (st, [C.POINTER(p), p, i32, i64, i32, i64, st, d, p, i32, d, i32, p, p,
                                         sz, p]),
            "splidar_plan_set_fluxes": (st, [p, fp, i32, p]),
            "splidar_plan_create_build": (st, [C.POINTER(p), fp, i32, st, st, p, i64, i64, p, i32, d, i32, p, p, sz,
                                               p]),
            "splidar_plan_execute": (st, [p, pinfo, p]),
            "splidar_plan_launch": (st, [p, p]),
            "splidar_plan_info": (st, [p, pinfo, p]),
            "splidar_plan_destroy": (None, [p]),
            "splidar_plan_kind": (C.c_int, [p]),
            "splidar_plan_gemv": (C.c_int, [p, p]),
            "splidar_plan_storage": (C.c_int, [p, p]),
            "splidar_plan_gemv_time": (st, [p, i32, C.POINTER(d), C.POINTER(i64), p]),
            "splidar_build_base_rows": (st, [fp, st, st, p, i64, i32, i32, p, sz, p]),
            "splidar_plan_create_rows": (st, [C.POINTER(p), p, i32, i32, i32, i64, st, d, p, i32, d, i32, p, p, p,
                                              sz, p]),
            "splidar_plan_shard_init": (st, [p, p]),
            "splidar_plan_shard_gemv": (st, [p, p]),
            "splidar_plan_shard_check": (st, [p, C.POINTER(i32), p]),
            "splidar_plan_shard_finish": (st, [p, pinfo, p]),
            "splidar_structured_workspace_bytes": (sz, [i32, i32, i32]),
            "splidar_stationary_structured": (st, [fp, i32, p, p, p, d, i32, p, p, sz, pinfo, p]),
            "splidar_second_eigenvalue": (st, [fp, i32, p, p, p, p, d, i32, p, sz, C.POINTER(SpectralInfo), p]),
            "splidar_spectral_dense_workspace_bytes": (sz, [i32]),
            "splidar_second_eigenvalue_dense": (st, [p, i32, i64, st, d, d, p, d, i32, p, sz,
                                                     C.POINTER(SpectralInfo), p]),
            "splidar_mixing_steps": (st, [fp, d, p, d, i32, p, C.POINTER(i32), p, sz, p]),
            "splidar_bin_trajectory": (st, [fp, d, p, i32, i32, p, p, p, sz, p]),
            "splidar_splan_create": (st, [C.POINTER(p), i32, fp, i32, p, p, p, d, i32, p, p, sz, p]),
            "splidar_splan_launch": (st, [p, p]),
            "splidar_splan_info": (st, [p, pinfo, C.POINTER(SpectralInfo), C.POINTER(C.c_float), p]),
            "splidar_splan_destroy": (None, [p]),
            "splidar_build_eq4": (st, [fp, d, st, p, i64, p]),
            "splidar_mc_workspace_bytes": (sz, [i32, i32]),
            "splidar_monte_carlo": (st, [fp, i32, p, p, p, C.c_uint64, i32, i32, i64, i64, i64, i32, p, i32, p, p,
                                         p, sz, p]),
            "splidar_strerror": (C.c_char_p, [st]),
            "splidar_last_cuda_error": (C.c_int, []),
            "splidar_build_info": (C.c_char_p, []),
        }
        for name, (res, args) in sig.items():
            fn = getattr(lib, name)
            fn.restype, fn.argtypes = res, args
        _LIB = lib
    return _LIB


def lib_path() -> str:
    _lib()
    return LIB_PATH


def build_info() -> str:
    return _lib().splidar_build_info().decode()


def _check(status: int, where: str, allow=()):
    if status != OK and status not in allow:
        raise SplidarError(status, where)
    return status


_RAW_STREAM = getattr(torch._C, "_cuda_getCurrentRawStream", None)


def _stream(stream=None) -> int:
    if stream is not None:
        return stream.cuda_stream
    if _RAW_STREAM is not None:                 # the current stream's handle without a Stream object
        return _RAW_STREAM(torch.cuda.current_device())
    return torch.cuda.current_stream().cuda_stream


def _allocates_on_stream(fn):
    """Runs fn with `stream` (when given) as torch's current stream, so that every workspace, output
    and temporary fn allocates belongs to the stream its kernels are enqueued on: the caching
    allocator then never hands a temporary that kernels on `stream` still read to another stream's
    allocation after fn returns. (The position of `stream` is looked up once, not per call.)"""
    names = list(inspect.signature(fn).parameters)
    pos = names.index("stream")

    @functools.wraps(fn)
    def wrapper(*args, **kwargs):
        st = kwargs.get("stream") if len(args) <= pos else args[pos]
        if isinstance(st, torch.cuda.Stream):
            with torch.cuda.stream(st):
                return fn(*args, **kwargs)
        return fn(*args, **kwargs)
    return wrapper


class _FluxArg:
    """Marshals any object with t_r, n_bins, tau, sigma, signal, background into splidar_flux.
    Hashable (frozen) flux objects are marshalled once and reused (see _flux_arg)."""

    def __init__(self, flux):
        self.tau = np.ascontiguousarray(flux.tau, dtype=np.float64).reshape(-1)
        self.sigma = np.ascontiguousarray(flux.sigma, dtype=np.float64).reshape(-1)
        self.signal = np.ascontiguousarray(flux.signal, dtype=np.float64).reshape(-1)
        dp = C.POINTER(C.c_double)
        self.s = _Flux(float(flux.t_r), int(flux.n_bins), int(self.tau.size),
                       self.tau.ctypes.data_as(dp), self.sigma.ctypes.data_as(dp),
                       self.signal.ctypes.data_as(dp), float(flux.background))


def shift(t_r: float, n_bins: int, t_d: float) -> int:
    """l = ceil((t_d mod t_r) N / t_r) mod N (Thm 2)."""
    out = C.c_int32(0)
    _check(_lib().splidar_shift(float(t_r), int(n_bins), float(t_d), C.byref(out)), "splidar_shift")
    return out.value


_FLUX_CACHE: dict = {}


def _flux_arg(flux) -> "_FluxArg":
    params = getattr(flux, "__dataclass_params__", None)
    if params is None or not params.frozen:             # only immutable fluxes are marshalled once
        return _FluxArg(flux)
    fa = _FLUX_CACHE.get(flux)
    if fa is None:
        if len(_FLUX_CACHE) > 4096:
            _FLUX_CACHE.clear()
        fa = _FLUX_CACHE[flux] = _FluxArg(flux)
    return fa


@functools.lru_cache(maxsize=1024)
def workspace_bytes(n_bins: int, n_matrices: int = 1, n_vectors: int = 1) -> int:
    return int(_lib().splidar_workspace_bytes(int(n_bins), int(n_matrices), int(n_vectors)))


def workspace(n_bins: int, n_matrices: int = 1, n_vectors: int = 1, device=None) -> torch.Tensor:
    n = workspace_bytes(n_bins, n_matrices, n_vectors)
    if n == 0:
        raise SplidarError(EINVAL, "splidar_workspace_bytes")
    t = torch.empty(n + 256, dtype=torch.uint8, device=device or "cuda")
    off = (-t.data_ptr()) % 256
    return t[off:off + n]


_SCRATCH: dict = {}


def _scratch_workspace(n_bins: int, n_matrices: int, n_vectors: int, device, stream) -> torch.Tensor:
    """The workspace of a one-shot solve when the caller passes none: kept per (device, stream, sizes)
    and reused, so repeated calls allocate nothing and hit the library's plan cache (which keys on
    the workspace pointer). Calls on different streams never share one."""
    dev = device if isinstance(device, torch.device) else (
        torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device()))
    key = (dev.index, _stream(stream), n_bins, n_matrices, n_vectors)
    ws = _SCRATCH.get(key)
    if ws is None:
        if len(_SCRATCH) > 64:
            _SCRATCH.clear()
        ws = _SCRATCH[key] = workspace(n_bins, n_matrices, n_vectors, device=dev)
    return ws


def leading_dim(n_bins: int, dtype=torch.float64) -> int:
    """Smallest ld >= N with ld * sizeof(dtype) a multiple of 16 bytes."""
    q = 16 // torch.tensor([], dtype=dtype).element_size()
    return (n_bins + q - 1) // q * q


def empty_matrix(n_bins: int, dtype=torch.float64, n_matrices: int | None = None, device=None) -> torch.Tensor:
    """Device matrix storage [N, ld] (or [M, N, ld]) returned as the [.., N, N] view."""
    ld = leading_dim(n_bins, dtype)
    shape = (n_bins, ld) if n_matrices is None else (n_matrices, n_bins, ld)
    return torch.empty(shape, dtype=dtype, device=device or "cuda")[..., :n_bins]


def _matrix_args(P: torch.Tensor):
    if not P.is_cuda or P.dtype not in _DTYPES or P.stride(-1) != 1:
        raise SplidarError(EINVAL, "matrix argument (CUDA fp64/fp32 row-major tensor expected)")
    return P.data_ptr(), P.shape[-1], P.stride(-2), _DTYPES[P.dtype]


@_allocates_on_stream
def flux_vectors(flux, ws: torch.Tensor | None = None, stream=None) -> dict:
    """Step 1 on the device: F(s_j), lambda(s_j), w_j, 1/D_j and Lambda (fp64 device tensors)."""
    N = int(flux.n_bins)
    ws = ws if ws is not None else workspace(N)
    F, lam, w, invd = (torch.empty(N, dtype=torch.float64, device=ws.device) for _ in range(4))
    L = torch.empty(1, dtype=torch.float64, device=ws.device)
    fa = _flux_arg(flux)
    _check(_lib().splidar_flux_vectors(C.byref(fa.s), F.data_ptr(), lam.data_ptr(), w.data_ptr(), invd.data_ptr(),
                                       L.data_ptr(), ws.data_ptr(), ws.numel(), _stream(stream)),
           "splidar_flux_vectors")
    return {"F": F, "lam": lam, "w": w, "inv_d": invd, "Lambda": L}


@_allocates_on_stream
def build_base(flux, dtype=torch.float64, mode: str = "factored", out: torch.Tensor | None = None,
               ws: torch.Tensor | None = None, stream=None) -> torch.Tensor:
    """Step 2: P~0 (N x N view of [N, ld] storage) on the current CUDA device (async)."""
    N = int(flux.n_bins)
    P = out if out is not None else empty_matrix(N, dtype)
    ptr, n, ld, dt = _matrix_args(P)
    ws = ws if ws is not None else workspace(N)
    fa = _flux_arg(flux)
    _check(_lib().splidar_build_base(C.byref(fa.s), dt, _MODES[mode], ptr, ld, ws.data_ptr(), ws.numel(),
                                     _stream(stream)), "splidar_build_base")
    return P


@_allocates_on_stream
def build_base_batched(fluxes, dtype=torch.float64, mode: str = "factored", out: torch.Tensor | None = None,
                       ws: torch.Tensor | None = None, stream=None) -> torch.Tensor:
    """Step 2 for M fluxes sharing N: P~0 [M, N, N] view of [M, N, ld] storage (async)."""
    M = len(fluxes)
    N = int(fluxes[0].n_bins)
    P = out if out is not None else empty_matrix(N, dtype, n_matrices=M)
    ptr, n, ld, dt = _matrix_args(P)
    ws = ws if ws is not None else workspace(N, M)
    fas = [_flux_arg(f) for f in fluxes]
    arr = (_Flux * M)(*[fa.s for fa in fas])
    _check(_lib().splidar_build_base_batched(arr, M, dt, _MODES[mode], ptr, ld, P.stride(0), ws.data_ptr(),
                                             ws.numel(), _stream(stream)), "splidar_build_base_batched")
    return P


@_allocates_on_stream
def build_eq4(flux, t_d: float, dtype=torch.float64, out: torch.Tensor | None = None, stream=None) -> torch.Tensor:
    """P~ element by element from Eq. 4 (the construction Theorem 2 replaces), async."""
    N = int(flux.n_bins)
    P = out if out is not None else empty_matrix(N, dtype)
    ptr, n, ld, dt = _matrix_args(P)
    fa = _flux_arg(flux)
    _check(_lib().splidar_build_eq4(C.byref(fa.s), float(t_d), dt, ptr, ld, _stream(stream)), "splidar_build_eq4")
    return P


@_allocates_on_stream
def apply_deadtime(P0: torch.Tensor, t_r: float, t_d: float, out: torch.Tensor | None = None,
                   stream=None) -> torch.Tensor:
    """Step 3 materialised: P[i] = P0[(i + l) mod N] (async)."""
    ptr, n, ld, dt = _matrix_args(P0)
    P = out if out is not None else empty_matrix(n, P0.dtype)
    optr, on, old, odt = _matrix_args(P)
    if old != ld or odt != dt or on != n:
        raise SplidarError(EINVAL, "apply_deadtime: out must match P0's N, ld and dtype")
    _check(_lib().splidar_apply_deadtime(ptr, optr, n, ld, dt, float(t_r), float(t_d), _stream(stream)),
           "splidar_apply_deadtime")
    return P


@_allocates_on_stream
def stationary(P0: torch.Tensor, t_r: float, t_d: float, tol: float = 1e-12, max_iter: int = 10 ** 6,
               out: torch.Tensor | None = None, ws: torch.Tensor | None = None, stream=None,
               check: bool = True):
    """Step 4: pi with pi (J_l P~0) = pi by on-device power iteration. Returns (pi, info dict)."""
    ptr, n, ld, dt = _matrix_args(P0)
    pi = out if out is not None else torch.empty(n, dtype=torch.float64, device=P0.device)
    ws = ws if ws is not None else _scratch_workspace(n, 1, 1, P0.device, stream)
    info = SolveInfo()
    st = _lib().splidar_stationary(ptr, n, ld, dt, float(t_r), float(t_d), float(tol), int(max_iter),
                                   pi.data_ptr(), ws.data_ptr(), ws.numel(), C.byref(info), _stream(stream))
    _check(st, "splidar_stationary", allow=() if check else (ENOCONV,))
    return pi, info.as_dict()


@_allocates_on_stream
def stationary_multi(P0: torch.Tensor, t_r: float, t_d, tol: float = 1e-12, max_iter: int = 10 ** 6,
                     out: torch.Tensor | None = None, ws: torch.Tensor | None = None, stream=None,
                     check: bool = True, out_host: torch.Tensor | None = None):
    """Step 4 for M matrices ([M, N, N] view) x V dead times each (t_d [M, V]) in one call; the
    instantiated solver is cached in the library per (buffers, sizes) and replayed by repeated calls.
    out_host (pinned CPU fp64 [M, V, N], optional) also receives pi within the same synchronisation.
    Returns (pi [M, V, N], list of M * V info dicts)."""
    ptr, n, ld, dt = _matrix_args(P0)
    M = P0.shape[0] if P0.dim() == 3 else 1
    mstride = P0.stride(0) if P0.dim() == 3 else n * ld
    T = np.ascontiguousarray(t_d, dtype=np.float64).reshape(M, -1)
    V = T.shape[1]
    pi = out if out is not None else torch.empty((M, V, n), dtype=torch.float64, device=P0.device)
    ws = ws if ws is not None else _scratch_workspace(n, M, V, P0.device, stream)
    infos = (SolveInfo * (M * V))()
    if out_host is not None and (out_host.is_cuda or out_host.dtype != torch.float64 or not out_host.is_contiguous()
                                 or out_host.numel() != M * V * n):
        raise SplidarError(EINVAL, "stationary_multi: out_host must be a contiguous CPU fp64 tensor of M*V*N")
    st = _lib().splidar_stationary_multi_host(ptr, M, mstride, n, ld, dt, float(t_r), T.ctypes.data, V, float(tol),
                                              int(max_iter), pi.data_ptr(),
                                              out_host.data_ptr() if out_host is not None else None,
                                              ws.data_ptr(), ws.numel(), infos, _stream(stream))
    _check(st, "splidar_stationary_multi", allow=() if check else (ENOCONV,))
    return pi, [i.as_dict() for i in infos]


def plan_cache_clear() -> None:
    """Destroy the library's cached one-shot solvers (splidar_plan_cache_clear)."""
    _lib().splidar_plan_cache_clear()


@_allocates_on_stream
def sweep(shape, S, B, t_d, dtype=torch.float64, mode: str = "factored", tol: float = 1e-12,
          max_iter: int = 10 ** 6, n_store: int | None = None, P0_store: torch.Tensor | None = None,
          ws: torch.Tensor | None = None, stream=None, check: bool = True, matrix_free: bool = False):
    """Steps 1-4 for (S[m], B[m], t_d[m]) items; shape.signal are relative pulse weights.
    matrix_free=True: no P~0 is stored (splidar_sweep with P0_store = NULL: the structured operator).
    Returns (pi [M, N] fp64 device tensor, list of info dicts)."""
    S = np.ascontiguousarray(S, dtype=np.float64).reshape(-1)
    B = np.ascontiguousarray(B, dtype=np.float64).reshape(-1)
    T = np.ascontiguousarray(t_d, dtype=np.float64).reshape(-1)
    M = S.size
    if B.size != M or T.size != M:
        raise SplidarError(EINVAL, "sweep: S, B, t_d must have equal length")
    N = int(shape.n_bins)
    if matrix_free:
        n_unique = len({(float(s), float(b)) for s, b in zip(S, B)})
        ws = ws if ws is not None else structured_workspace(N, n_unique, M)
        pi = torch.empty((M, N), dtype=torch.float64, device=ws.device)
        infos = (SolveInfo * M)()
        fa = _flux_arg(shape)
        st = _lib().splidar_sweep(C.byref(fa.s), M, S.ctypes.data, B.ctypes.data, T.ctypes.data, F64,
                                  _MODES[mode], float(tol), int(max_iter), pi.data_ptr(), None, 0, 0,
                                  ws.data_ptr(), ws.numel(), infos, _stream(stream))
        _check(st, "splidar_sweep", allow=() if check else (ENOCONV,))
        return pi, [i.as_dict() for i in infos]
    n_unique = len({(float(s), float(b)) for s, b in zip(S, B)})
    if P0_store is None:
        n_store = n_store or n_unique
        P0_store = empty_matrix(N, dtype, n_matrices=n_store)
    else:
        n_store = P0_store.shape[0] if P0_store.dim() == 3 else 1
    ptr, n, ld, dt = _matrix_args(P0_store)
    if ws is None:
        max_items = 1
        counts = {}
        for s, b in zip(S, B):
            counts[(float(s), float(b))] = counts.get((float(s), float(b)), 0) + 1
        max_items = min(MAX_VECTORS, max(counts.values()))
        ws = workspace(N, min(n_store, n_unique), max_items, device=P0_store.device)
    pi = torch.empty((M, N), dtype=torch.float64, device=P0_store.device)
    infos = (SolveInfo * M)()
    fa = _flux_arg(shape)
    st = _lib().splidar_sweep(C.byref(fa.s), M, S.ctypes.data, B.ctypes.data, T.ctypes.data, dt, _MODES[mode],
                              float(tol), int(max_iter), pi.data_ptr(), ptr, int(n_store), ld, ws.data_ptr(),
                              ws.numel(), infos, _stream(stream))
    _check(st, "splidar_sweep", allow=() if check else (ENOCONV,))
    return pi, [i.as_dict() for i in infos]


class Plan:
    """An instantiated CUDA-graph power-iteration solver for M matrices x V dead times.

    P0: [N, N] or [M, N, N] view (row-major, ld = stride); t_d: array [M, V]. pi: [M, V, N] fp64.
    execute() reruns the solve from pi^0 and returns the infos; launch() only enqueues."""

    def __init__(self, P0: torch.Tensor, t_r: float, t_d, tol: float = 1e-12, max_iter: int = 10 ** 6,
                 ws: torch.Tensor | None = None, stream=None, build=None, mode: str = "factored"):
        """build: fluxes (one per matrix) -> every launch also builds P0 (splidar_plan_create_build):
        steps 1-2 and the column sums that give iteration 1 without a GEMV pass."""
        ptr, n, ld, dt = _matrix_args(P0)
        M = P0.shape[0] if P0.dim() == 3 else 1
        mstride = P0.stride(0) if P0.dim() == 3 else n * ld
        T = np.ascontiguousarray(t_d, dtype=np.float64).reshape(M, -1)
        V = T.shape[1]
        self.M, self.V, self.N = M, V, n
        self.P0 = P0
        self.pi = torch.empty((M, V, n), dtype=torch.float64, device=P0.device)
        self.ws = ws if ws is not None else workspace(n, M, V, device=P0.device)
        self._T = T
        self._h = C.c_void_p(None)
        if build is not None:
            fl = list(build) if isinstance(build, (list, tuple)) else [build]
            if len(fl) != M:
                raise SplidarError(EINVAL, "Plan(build=...): one flux per matrix")
            self._fas = [_flux_arg(f) for f in fl]
            arr = (_Flux * M)(*[fa.s for fa in self._fas])
            self._farr = arr
            _check(_lib().splidar_plan_create_build(C.byref(self._h), arr, M, _MODES[mode], dt, ptr, mstride, ld,
                                                    T.ctypes.data, V, float(tol), int(max_iter), self.pi.data_ptr(),
                                                    self.ws.data_ptr(), self.ws.numel(), _stream(stream)),
                   "splidar_plan_create_build")
            return
        _check(_lib().splidar_plan_create(C.byref(self._h), ptr, M, mstride, n, ld, dt, float(t_r), T.ctypes.data,
                                          V, float(tol), int(max_iter), self.pi.data_ptr(), self.ws.data_ptr(),
                                          self.ws.numel(), _stream(stream)), "splidar_plan_create")

    def launch(self, stream=None):
        _check(_lib().splidar_plan_launch(self._h, _stream(stream)), "splidar_plan_launch")

    def set_fluxes(self, fluxes, stream=None):
        """New theta for a building plan (Plan(build=...)): same N and t_r, one flux per matrix."""
        fl = list(fluxes) if isinstance(fluxes, (list, tuple)) else [fluxes]
        fas = [_flux_arg(f) for f in fl]
        key = tuple(id(fa) for fa in fas)          # the marshalled array of the last call, reused
        last = getattr(self, "_flux_arr", None)
        if last is not None and last[0] == key:
            arr = last[1]
        else:
            arr = (_Flux * len(fl))(*[fa.s for fa in fas])
            self._flux_arr = (key, arr, fas)       # fas keeps the parameter arrays arr points into alive
        _check(_lib().splidar_plan_set_fluxes(self._h, arr, len(fl), _stream(stream)), "splidar_plan_set_fluxes")

    @property
    def fused(self) -> bool:
        """True when the plan is one clustered launch (N <= 2048), capturable into a CUDA graph."""
        return _lib().splidar_plan_kind(self._h) == 1

    KINDS = {0: "graph", 1: "fused", 2: "loop"}

    @property
    def kind(self) -> str:
        """'fused' (N <= 2048, one clustered launch), 'loop' (a graph whose iterations are one cooperative
        launch of the persistent GEMV + check kernel) or 'graph' (GEMV + check in a conditional WHILE node)."""
        return self.KINDS[_lib().splidar_plan_kind(self._h)]

    GEMV_NAMES = {0: "fused", 1: "fp64", 2: "tensor_i8"}

    def gemv(self, stream=None) -> str:
        """The GEMV kernel of the last launch: 'tensor_i8' (tcgen05 int8 split), 'fp64' (DMMA / DFMA)
        or 'fused' (small-N single launch). Synchronises the stream."""
        k = _lib().splidar_plan_gemv(self._h, _stream(stream))
        if k < 0:
            raise SplidarError(ECUDA, "splidar_plan_gemv")
        return self.GEMV_NAMES[k]

    def gemv_time(self, reset: bool = False, stream=None):
        """(seconds, launches) of the plan's GEMV kernel since the last reset, measured on the device
        (splidar_plan_gemv_time). Synchronises the stream."""
        sec, n = C.c_double(0.0), C.c_int64(0)
        _check(_lib().splidar_plan_gemv_time(self._h, int(reset), C.byref(sec), C.byref(n), _stream(stream)),
               "splidar_plan_gemv_time")
        return sec.value, n.value

    def storage(self, stream=None) -> str:
        """The form of P0 after the last launch: 'ieee' or 'encoded' (a building plan's per-column
        scaled integers, splidar_plan_create_build). Synchronises the stream."""
        k = _lib().splidar_plan_storage(self._h, _stream(stream))
        if k < 0:
            raise SplidarError(ECUDA, "splidar_plan_storage")
        return ("ieee", "encoded")[k]

    def info(self, stream=None, check: bool = True) -> list:
        infos = (SolveInfo * (self.M * self.V))()
        st = _lib().splidar_plan_info(self._h, infos, _stream(stream))
        _check(st, "splidar_plan_info", allow=() if check else (ENOCONV,))
        return [i.as_dict() for i in infos]

    def execute(self, stream=None, check: bool = True) -> list:
        self.launch(stream)
        return self.info(stream, check)

    def close(self):
        if self._h:
            _lib().splidar_plan_destroy(self._h)
            self._h = C.c_void_p(None)

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


@_allocates_on_stream
def build_base_rows(flux, row0: int, n_rows: int, dtype=torch.float64, mode: str = "factored",
                    out: torch.Tensor | None = None, ws: torch.Tensor | None = None, stream=None) -> torch.Tensor:
    """Rows [row0, row0 + n_rows) of P~0 ([n_rows, N] view of [n_rows, ld] storage), the same entries
    as those rows of build_base (SURVEY §8(e)(ii) row shard)."""
    N = int(flux.n_bins)
    ld = leading_dim(N, dtype)
    P = out if out is not None else torch.empty((n_rows, ld), dtype=dtype, device="cuda")[:, :N]
    ptr, n, ldp, dt = _matrix_args(P)
    ws = ws if ws is not None else workspace(N)
    fa = _flux_arg(flux)
    _check(_lib().splidar_build_base_rows(C.byref(fa.s), dt, _MODES[mode], ptr, ldp, int(row0), int(n_rows),
                                          ws.data_ptr(), ws.numel(), _stream(stream)), "splidar_build_base_rows")
    return P


class ShardPlan:
    """One rank's part of a row-sharded power iteration (include/splidar.h): P0_rows
    holds rows [row0, row0 + n_rows) of the N x N P~0; t_d: V dead times. ypart [V, N] is this rank's
    partial product, to be summed over the ranks between gemv() and check(); pi [V, N] after finish().
    See shard.sharded_solve for the loop."""

    def __init__(self, P0_rows: torch.Tensor, row0: int, n_bins: int, t_r: float, t_d, tol: float = 1e-12,
                 max_iter: int = 10 ** 6, ws: torch.Tensor | None = None, stream=None):
        ptr, n, ld, dt = _matrix_args(P0_rows)
        if n != n_bins:
            raise SplidarError(EINVAL, "ShardPlan: P0_rows must have N columns")
        T = np.ascontiguousarray(t_d, dtype=np.float64).reshape(-1)
        self.V, self.N, self.stream = T.size, n_bins, stream
        self.pi = torch.empty((self.V, n_bins), dtype=torch.float64, device=P0_rows.device)
        self.ypart = torch.zeros((self.V, n_bins), dtype=torch.float64, device=P0_rows.device)
        self.ws = ws if ws is not None else workspace(n_bins, 1, self.V, device=P0_rows.device)
        self.P0_rows, self._T = P0_rows, T
        self._h = C.c_void_p(None)
        _check(_lib().splidar_plan_create_rows(C.byref(self._h), ptr, int(row0), int(P0_rows.shape[0]), n_bins, ld,
                                               dt, float(t_r), T.ctypes.data, self.V, float(tol), int(max_iter),
                                               self.pi.data_ptr(), self.ypart.data_ptr(), self.ws.data_ptr(),
                                               self.ws.numel(), _stream(stream)), "splidar_plan_create_rows")

    def init(self):
        _check(_lib().splidar_plan_shard_init(self._h, _stream(self.stream)), "splidar_plan_shard_init")

    def gemv(self):
        _check(_lib().splidar_plan_shard_gemv(self._h, _stream(self.stream)), "splidar_plan_shard_gemv")

    def check(self) -> bool:
        more = C.c_int32(0)
        _check(_lib().splidar_plan_shard_check(self._h, C.byref(more), _stream(self.stream)),
               "splidar_plan_shard_check")
        return bool(more.value)

    def finish(self, check: bool = True) -> list:
        infos = (SolveInfo * self.V)()
        st = _lib().splidar_plan_shard_finish(self._h, infos, _stream(self.stream))
        _check(st, "splidar_plan_shard_finish", allow=() if check else (ENOCONV,))
        return [i.as_dict() for i in infos]

    def close(self):
        if self._h:
            _lib().splidar_plan_destroy(self._h)
            self._h = C.c_void_p(None)

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


@dataclass
class HostResult:
    pi: np.ndarray
    info: dict


def solve_host(flux, t_d: float, dtype=torch.float64, mode: str = "factored", tol: float = 1e-12,
               max_iter: int = 10 ** 6, P0: torch.Tensor | None = None, ws: torch.Tensor | None = None,
               pi_host: torch.Tensor | None = None) -> HostResult:
    """End-to-end public call with host inputs and host output: theta (host) -> device build of P~0
    -> on-device power iteration -> pi copied into (pinned) host memory."""
    N = int(flux.n_bins)
    P0 = build_base(flux, dtype, mode, out=P0, ws=ws)
    pi, info = stationary(P0, flux.t_r, t_d, tol, max_iter, ws=ws)
    if pi_host is None:
        pi_host = torch.empty(N, dtype=torch.float64, pin_memory=True)
    pi_host.copy_(pi, non_blocking=True)
    torch.cuda.current_stream().synchronize()
    return HostResult(pi_host.numpy(), info)


# ------------------------------------------------------------------ structured operator (f1, f2)
def structured_workspace(n_bins: int, n_profiles: int = 1, n_items: int = 1, device=None) -> torch.Tensor:
    n = int(_lib().splidar_structured_workspace_bytes(int(n_bins), int(n_profiles), int(n_items)))
    if n == 0:
        raise SplidarError(EINVAL, "splidar_structured_workspace_bytes")
    t = torch.empty(n + 256, dtype=torch.uint8, device=device or "cuda")
    off = (-t.data_ptr()) % 256
    return t[off:off + n]


def _items(shape, S, B, t_d):
    S = np.ascontiguousarray(S, dtype=np.float64).reshape(-1)
    B = np.ascontiguousarray(B, dtype=np.float64).reshape(-1)
    T = np.ascontiguousarray(t_d, dtype=np.float64).reshape(-1)
    if B.size != S.size or T.size != S.size or S.size < 1:
        raise SplidarError(EINVAL, "S, B, t_d must have equal non-zero length")
    # distinct (S, B) pairs, compared numerically as the library groups them: the workspace size
    n_prof = int(np.unique(S + 1j * B).size)
    return S, B, T, n_prof


def _records(ctypes_array) -> np.ndarray:
    """Per-item infos as a numpy structured array (a zero-copy view of the ctypes array; fields as the
    C struct: infos[m]["iters"], infos["converged"], ...). Used by the batched structured calls, whose
    item counts make a list of dicts the dominant host cost."""
    return np.ctypeslib.as_array(ctypes_array)


def lambda2_of(rec) -> complex:
    """lambda_2 of one spectral record (lambda2_re + i lambda2_im)."""
    return complex(float(rec["lambda2_re"]), float(rec["lambda2_im"]))


@_allocates_on_stream
def stationary_structured(shape, S, B, t_d, tol: float = 1e-12, max_iter: int = 10 ** 6,
                          ws: torch.Tensor | None = None, stream=None, check: bool = True):
    """f2: pi for (S[m], B[m], t_d[m]) items by power iteration on the matrix-free operator (no P~0 is
    stored). shape.signal are relative pulse weights (as sweep). Returns (pi [M, N] fp64, infos)."""
    S, B, T, n_prof = _items(shape, S, B, t_d)
    M, N = S.size, int(shape.n_bins)
    ws = ws if ws is not None else structured_workspace(N, n_prof, M)
    pi = torch.empty((M, N), dtype=torch.float64, device=ws.device)
    infos = (SolveInfo * M)()
    fa = _flux_arg(shape)
    st = _lib().splidar_stationary_structured(C.byref(fa.s), M, S.ctypes.data, B.ctypes.data, T.ctypes.data,
                                              float(tol), int(max_iter), pi.data_ptr(), ws.data_ptr(), ws.numel(),
                                              infos, _stream(stream))
    _check(st, "splidar_stationary_structured", allow=() if check else (ENOCONV,))
    return pi, _records(infos)


@_allocates_on_stream
def second_eigenvalue(shape, S, B, t_d, pi: torch.Tensor, tol: float = 1e-13, max_iter: int = 10 ** 5,
                      ws: torch.Tensor | None = None, stream=None, check: bool = True) -> list:
    """f1: lambda_2 of P~ per item (modulus, phase in [0, pi], gap); pi = the items' stationary vectors
    [M, N] on the device. Returns a numpy structured array with the fields of SpectralInfo
    (lambda2_of(rec) gives the complex value)."""
    S, B, T, n_prof = _items(shape, S, B, t_d)
    M, N = S.size, int(shape.n_bins)
    if not pi.is_cuda or pi.dtype != torch.float64 or pi.numel() != M * N or not pi.is_contiguous():
        raise SplidarError(EINVAL, "second_eigenvalue: pi must be a contiguous CUDA fp64 [M, N] tensor")
    ws = ws if ws is not None else structured_workspace(N, n_prof, M, device=pi.device)
    infos = (SpectralInfo * M)()
    fa = _flux_arg(shape)
    st = _lib().splidar_second_eigenvalue(C.byref(fa.s), M, S.ctypes.data, B.ctypes.data, T.ctypes.data,
                                          pi.data_ptr(), float(tol), int(max_iter), ws.data_ptr(), ws.numel(),
                                          infos, _stream(stream))
    _check(st, "splidar_second_eigenvalue", allow=() if check else (ENOCONV,))
    return _records(infos)


@_allocates_on_stream
def second_eigenvalue_dense(P0: torch.Tensor, t_r: float, t_d: float, pi: torch.Tensor, tol: float = 1e-13,
                            max_iter: int = 10 ** 5, ws: torch.Tensor | None = None, stream=None,
                            check: bool = True) -> dict:
    """f1 on a stored matrix: lambda_2 of P~ = J_l P0 (any row-stochastic P0 [N, >= N] fp64/fp32 on the
    device, l from (t_r, t_d)); pi = the stationary vector of P~ [N] fp64 on the device. Every product
    is a pass of the multi-vector GEMV over P0. Returns a dict with the fields of SpectralInfo."""
    ptr, n, ld, dt = _matrix_args(P0)
    if not pi.is_cuda or pi.dtype != torch.float64 or pi.numel() != n or not pi.is_contiguous():
        raise SplidarError(EINVAL, "second_eigenvalue_dense: pi must be a contiguous CUDA fp64 [N] tensor")
    if ws is None:
        nb = _lib().splidar_spectral_dense_workspace_bytes(n)
        t = torch.empty(nb + 256, dtype=torch.uint8, device=P0.device)
        off = (-t.data_ptr()) % 256
        ws = t[off:off + nb]
    info = SpectralInfo()
    st = _lib().splidar_second_eigenvalue_dense(ptr, n, ld, dt, float(t_r), float(t_d), pi.data_ptr(), float(tol),
                                                int(max_iter), ws.data_ptr(), ws.numel(), C.byref(info),
                                                _stream(stream))
    _check(st, "splidar_second_eigenvalue_dense", allow=() if check else (ENOCONV,))
    return info.as_dict()


@_allocates_on_stream
def mixing_steps(flux, t_d: float, pi: torch.Tensor, eps: float = 1e-3, max_steps: int = 10 ** 5,
                 ws: torch.Tensor | None = None, stream=None, check: bool = True):
    """f1: smallest n with max_i 1/2 ||e_i P~^n - pi||_1 <= eps. Returns (n, per-start n_i int32 tensor)."""
    N = int(flux.n_bins)
    if not pi.is_cuda or pi.dtype != torch.float64 or pi.numel() != N or not pi.is_contiguous():
        raise SplidarError(EINVAL, "mixing_steps: pi must be a contiguous CUDA fp64 [N] tensor")
    ws = ws if ws is not None else structured_workspace(N, 1, N, device=pi.device)
    per = torch.empty(N, dtype=torch.int32, device=pi.device)
    out = C.c_int32(0)
    fa = _flux_arg(flux)
    st = _lib().splidar_mixing_steps(C.byref(fa.s), float(t_d), pi.data_ptr(), float(eps), int(max_steps),
                                     per.data_ptr(), C.byref(out), ws.data_ptr(), ws.numel(), _stream(stream))
    _check(st, "splidar_mixing_steps", allow=() if check else (ENOCONV,))
    return out.value, per


@_allocates_on_stream
def bin_trajectory(flux, t_d: float, start: torch.Tensor, bin: int, steps: int, ws: torch.Tensor | None = None,
                   stream=None):
    """f1: (start P~^n)[bin] for n = 0..steps. Returns (traj [steps + 1], start P~^steps [N])."""
    N = int(flux.n_bins)
    if not start.is_cuda or start.dtype != torch.float64 or start.numel() != N or not start.is_contiguous():
        raise SplidarError(EINVAL, "bin_trajectory: start must be a contiguous CUDA fp64 [N] tensor")
    ws = ws if ws is not None else structured_workspace(N, 1, 1, device=start.device)
    traj = torch.empty(int(steps) + 1, dtype=torch.float64, device=start.device)
    fin = torch.empty(N, dtype=torch.float64, device=start.device)
    fa = _flux_arg(flux)
    _check(_lib().splidar_bin_trajectory(C.byref(fa.s), float(t_d), start.data_ptr(), int(bin), int(steps),
                                         traj.data_ptr(), fin.data_ptr(), ws.data_ptr(), ws.numel(),
                                         _stream(stream)), "splidar_bin_trajectory")
    return traj, fin


def flux_items(flux):
    """(shape, S, B) for one flux in the items convention: shape = flux, S = 1, B = flux.background."""
    return flux, np.array([1.0]), np.array([float(flux.background)])


class StructPlan:
    """Structured (matrix-free) solver plan: kind "solve" (f2, pi out) or "lambda2" (f1, pi in).
    launch() only enqueues (step-1 vectors + kernel); info() syncs and returns (infos, kernel_ms)."""

    def __init__(self, kind: str, shape, S, B, t_d, pi: torch.Tensor | None = None, tol: float | None = None,
                 max_iter: int | None = None, ws: torch.Tensor | None = None, stream=None):
        S, B, T, n_prof = _items(shape, S, B, t_d)
        self.kind = {"solve": 0, "lambda2": 1}[kind]
        self.M, self.N = S.size, int(shape.n_bins)
        if tol is None:
            tol = 1e-12 if self.kind == 0 else 1e-13
        if max_iter is None:
            max_iter = 10 ** 6 if self.kind == 0 else 10 ** 5
        if self.kind == 0 and pi is None:
            pi = torch.empty((self.M, self.N), dtype=torch.float64, device="cuda")
        if pi is None or not pi.is_cuda or pi.dtype != torch.float64 or pi.numel() != self.M * self.N:
            raise SplidarError(EINVAL, "StructPlan: pi must be a CUDA fp64 [M, N] tensor")
        self.pi = pi
        self.ws = ws if ws is not None else structured_workspace(self.N, n_prof, self.M, device=pi.device)
        self._keep = (S, B, T)
        self._h = C.c_void_p(None)
        fa = _flux_arg(shape)
        _check(_lib().splidar_splan_create(C.byref(self._h), self.kind, C.byref(fa.s), self.M, S.ctypes.data,
                                           B.ctypes.data, T.ctypes.data, float(tol), int(max_iter), pi.data_ptr(),
                                           self.ws.data_ptr(), self.ws.numel(), _stream(stream)),
               "splidar_splan_create")

    def launch(self, stream=None):
        _check(_lib().splidar_splan_launch(self._h, _stream(stream)), "splidar_splan_launch")

    def info(self, stream=None, check: bool = True):
        ms = C.c_float(0.0)
        if self.kind == 0:
            infos = (SolveInfo * self.M)()
            st = _lib().splidar_splan_info(self._h, infos, None, C.byref(ms), _stream(stream))
        else:
            infos = (SpectralInfo * self.M)()
            st = _lib().splidar_splan_info(self._h, None, infos, C.byref(ms), _stream(stream))
        _check(st, "splidar_splan_info", allow=() if check else (ENOCONV,))
        return _records(infos), float(ms.value)

    def close(self):
        if self._h:
            _lib().splidar_splan_destroy(self._h)
            self._h = C.c_void_p(None)

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


@_allocates_on_stream
def monte_carlo(shape, S, B, t_d, seed: int, n_runs: int, n_hist: int, n_burn: int = 100, n_regs: int = 0,
                n_cycles: int = 0, n_record: int = 0, n_split: int = 1, stream=None):
    """histograms [M, n_runs, n_hist] (int64 CUDA tensor) of simulated detection timestamps
     per item; with n_record > 0 also (q_rec, t_rec) [M * n_runs, n_record] of every chain."""
    S, B, T, n_prof = _items(shape, S, B, t_d)
    M = S.size
    hist = torch.empty((M, int(n_runs), int(n_hist)), dtype=torch.int64, device="cuda")
    nb = int(_lib().splidar_mc_workspace_bytes(n_prof, M))
    if nb == 0:
        raise SplidarError(EINVAL, "splidar_mc_workspace_bytes")
    ws = torch.empty(nb + 256, dtype=torch.uint8, device="cuda")
    ws = ws[(-ws.data_ptr()) % 256:][:nb]
    nr = max(0, int(n_record))
    q_rec = torch.empty((M * int(n_runs) * int(n_split), max(nr, 1)), dtype=torch.int64, device="cuda")
    t_rec = torch.empty((M * int(n_runs) * int(n_split), max(nr, 1)), dtype=torch.float64, device="cuda")
    fa = _flux_arg(shape)
    _check(_lib().splidar_monte_carlo(C.byref(fa.s), M, S.ctypes.data, B.ctypes.data, T.ctypes.data,
                                      int(seed) & (2 ** 64 - 1), int(n_runs), int(n_split), int(n_burn), int(n_regs),
                                      int(n_cycles), int(n_hist), hist.data_ptr(), nr,
                                      q_rec.data_ptr() if nr else None, t_rec.data_ptr() if nr else None,
                                      ws.data_ptr(), ws.numel(), _stream(stream)), "splidar_monte_carlo")
    if nr:
        return hist, q_rec, t_rec
    return hist
