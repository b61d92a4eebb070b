"""Test-side independent cross-check for large N (pin P11): the stationary vector of
J_l P~0 from the rank-1 semiseparable form of E_base, O(N) per iteration, computed in
long double from the ORACLE's pointwise lambda(s_j) and closed-form F(s_j). Shares nothing with the
CUDA path. Used where the dense oracle matrix would not fit or take minutes (N = 16384, 32768)."""
from __future__ import annotations

import math

import numpy as np

import oracle


def oracle_vectors(flux):
    N = flux.n_bins
    d = flux.t_r / N
    s = (np.arange(N) + 0.5) * d
    lam = np.array([oracle.lam(flux, t) for t in s], dtype=np.float64)
    F = np.array([oracle.F(flux, t) for t in s], dtype=np.float64)
    return lam, F, oracle.Lambda(flux)


def structured_pi(flux, t_d: float, tol: float = 1e-15, max_iter: int = 10000, vectors=None):
    lam, F, Lam = vectors if vectors is not None else oracle_vectors(flux)
    ld = np.longdouble
    w = lam.astype(ld) * np.exp(-F.astype(ld))
    eL = np.exp(-ld(Lam))
    U = np.cumsum(w[::-1])[::-1]
    L = np.concatenate([[ld(0)], np.cumsum(w)[:-1]])
    D = U + eL * L
    l = oracle.shift_l(flux, t_d)
    N = flux.n_bins
    pi = np.full(N, ld(1) / N)
    for it in range(1, max_iter + 1):
        z = np.roll(pi, l) / D           # x_r = pi[(r - l) mod N], divided by D_r
        c = np.cumsum(z)
        y = w * (c + eL * (c[-1] - c))
        y /= y.sum()
        ch = float(np.abs(y - pi).sum())
        pi = y
        if ch < tol:
            break
    return pi.astype(np.float64), it


def sampled_rows(flux, t_d: float, rows):
    return np.stack([oracle.rows_eq4(flux, t_d, int(r), int(r) + 1)[0] for r in rows])
