"""Property-based pins of the CPU oracle (hypothesis; CPU only). The fixed-case pins of
test_oracle_pins.py checked at randomly drawn theta = (t_r, N, K pulses (tau, sigma, S), B, t_d):
the shapes, sizes and value ranges of the paper's workloads, shrunk to N <= 48 so that every draw
builds Eq. 4 entry by entry in milliseconds. None re-types the oracle's formula: each property is a
consequence the paper or the mathematics fixes.

* P1 row-stochastic, strictly positive (B > 0): the normalisation of P:79 and an everywhere-positive
  flux.
* Theorem 2: P~(t_d) is P~(0) with its rows rolled by -l, l = ceil(x_d / Delta),
  x_d = t_d mod t_r; the opposite direction must fail whenever l != 0 mod N.
* Constant flux (S = 0, P:50 with only the background): the chain is invariant under a shift of the
  time axis by one bin, so P~ is circulant (P~[i+1][j+1] = P~[i][j], indices mod N), at every t_d.
* The stationary vector: the dense solve gives pi >= 0, sum 1, ||pi P~ - pi||_1 tiny, and the
  power iteration reaches the same vector.
"""
import numpy as np
import pytest
from hypothesis import HealthCheck, given, settings
from hypothesis import strategies as st

import oracle
from workloads import Flux

SETTINGS = settings(max_examples=40, deadline=None, suppress_health_check=[HealthCheck.function_scoped_fixture])


@st.composite
def thetas(draw, constant=False):
    t_r = draw(st.sampled_from([100.0, 200.0, 64.0, 37.5]))
    n = draw(st.integers(min_value=2, max_value=48))
    k = 0 if constant else draw(st.integers(min_value=0, max_value=2))
    d = t_r / n
    tau = tuple(draw(st.floats(0.0, t_r, exclude_max=True)) for _ in range(k))
    sigma = tuple(draw(st.floats(0.3 * d, 5.0 * d)) for _ in range(k))
    signal = tuple(draw(st.floats(0.0, 10.0)) for _ in range(k))
    background = draw(st.floats(1e-3, 5.0))
    # dead times: anywhere in three periods, plus whole bins and whole periods exactly
    m = draw(st.integers(min_value=0, max_value=3 * n))
    t_d = draw(st.one_of(st.floats(0.0, 3.0 * t_r), st.just(m * d), st.just(float(m % 4) * t_r)))
    return Flux(t_r, n, tau, sigma, signal, background), float(t_d)


@SETTINGS
@given(thetas())
def test_prop_row_stochastic_and_positive(oracle_lib, th):
    f, td = th
    P = oracle.build_eq4(f, td)
    assert P.shape == (f.n_bins, f.n_bins)
    assert np.all(np.isfinite(P)) and np.all(P > 0.0)
    assert np.max(np.abs(P.sum(axis=1) - 1.0)) <= 1e-12


@SETTINGS
@given(thetas())
def test_prop_theorem2_row_roll(oracle_lib, th):
    f, td = th
    n = f.n_bins
    P = oracle.build_eq4(f, td)
    P0 = oracle.build_eq4(f, 0.0)
    l = oracle.shift_l(f, td)
    assert 0 <= l <= n
    assert np.max(np.abs(np.roll(P0, -l, axis=0) - P)) <= 1e-15
    if l % n and np.max(np.abs(np.roll(P0, -l, axis=0) - np.roll(P0, +l, axis=0))) > 1e-12:
        assert np.max(np.abs(np.roll(P0, +l, axis=0) - P)) > 1e-13


@SETTINGS
@given(thetas(constant=True))
def test_prop_constant_flux_circulant(oracle_lib, th):
    f, td = th
    P = oracle.build_eq4(f, td)
    shifted = np.roll(np.roll(P, 1, axis=0), 1, axis=1)     # shifted[i][j] = P[i-1][j-1]
    assert np.max(np.abs(shifted - P)) <= 1e-14


@SETTINGS
@given(thetas())
def test_prop_stationary_vector(oracle_lib, th):
    f, td = th
    P = oracle.build_eq4(f, td)
    pi = oracle.stationary_dense(P)
    assert np.all(pi >= -1e-15) and abs(pi.sum() - 1.0) <= 1e-13
    assert np.sum(np.abs(pi @ P - pi)) <= 1e-13
    pw, _, _, ok = oracle.stationary_power(P, 1e-14)
    if ok:
        assert np.sum(np.abs(pw - pi)) <= 1e-9
