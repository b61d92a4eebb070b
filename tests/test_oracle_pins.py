"""Pins of the CPU oracle against what the paper and the mathematics fix (CPU only).

Each test names the pin of DESIGN.md §4 / SURVEY §8(c) it implements and the passage it follows.
None of these re-type the oracle's formula: they use closed forms derived independently
(constant flux, two-state chains, exact rationals), invariants, limits, numerical quadrature,
an independent O(N) algorithm and a continuous-time Monte Carlo of the physical process.
"""
import math
from fractions import Fraction

import numpy as np
import pytest
from scipy import integrate

import oracle
from workloads import Flux, config, random_flux

RNG_SEED = 20250920


def _rand_cases(n_cases, n_bins, seed=RNG_SEED):
    rng = np.random.default_rng(seed)
    out = []
    for c in range(n_cases):
        f = random_flux(rng, n_bins, 1 + c % 2)
        out.append((f, float(rng.uniform(0.0, 3.0 * f.t_r))))
    return out


# ---------------------------------------------------------------- P1 row-stochastic
@pytest.mark.parametrize("f,td", _rand_cases(4, 96))
def test_p1_row_stochastic(oracle_lib, f, td):
    P = oracle.build_eq4(f, td)
    assert np.all(P > 0.0)                                   # B > 0 => every transition possible
    assert np.max(np.abs(P.sum(axis=1) - 1.0)) <= 1e-12


# ------------------------------------------- P2 permuted base == direct Eq. 4 (Thm 2)
@pytest.mark.parametrize("f,td", _rand_cases(6, 80, seed=3) + [(config(1).items[0].flux, 75.0)])
def test_p2_row_permutation_equals_direct(oracle_lib, f, td):
    """Row i of P~(t_d) is row (i + l) mod N of P~(0), l = ceil(x_d / Delta).
    Exact after normalisation, so the tolerance is rounding only; the opposite roll
    direction must fail."""
    P = oracle.build_eq4(f, td)
    P0 = oracle.build_eq4(f, 0.0)
    l = oracle.shift_l(f, td)
    assert np.max(np.abs(np.roll(P0, -l, axis=0) - P)) <= 1e-15
    if l % f.n_bins:
        assert np.max(np.abs(np.roll(P0, +l, axis=0) - P)) > 1e-6


# ------------------------------- P3 raw dead time in the bounds, whole periods (Eq. 4)
def _raw_bound_integral(f, i, j, t_d):
    """The physical definition: a registration at s_i re-arms the SPAD at the RAW time
    a = s_i + t_d on the unrolled time line; the next registration in bin j happens at the first
    later visit b = ceil((a - s_j) / t_r) t_r + s_j of s_j (Eq. 3's upper limit with the raw a,
    P:102), and Eq. 4 discretises the lower limit to D(a) = (ceil(a / Delta) - 1/2) Delta.
    Returns int_{D(a)}^{b} lambda~ by quadrature over however many periods [D(a), b] spans -- no
    fmod of t_d anywhere, so a wrong period reduction in the oracle cannot cancel out."""
    # the two ceilings in exact rational arithmetic (t_d and t_r are exact binary fractions), so a
    # bound that lands exactly on a bin centre (t_d a whole number of periods) is not pushed a
    # period further by rounding; the limits themselves are then plain floats
    d = Fraction(f.t_r) / f.n_bins
    a = (i + Fraction(1, 2)) * d + Fraction(t_d)
    s_j = (j + Fraction(1, 2)) * d
    Da = float((math.ceil(a / d) - Fraction(1, 2)) * d)
    b = float(math.ceil((a - s_j) / Fraction(f.t_r)) * Fraction(f.t_r) + s_j)
    return _lam_tilde_integral(f, Da, b)


@pytest.mark.parametrize("m", [1, 2, 3])
def test_p3_raw_dead_time_and_whole_periods(oracle_lib, m):
    """t_d = m t_r + x (m = 1..3): every unnormalised oracle entry equals lambda(s_j) exp(-I) with
    I the quadrature of lambda~ between the RAW-dead-time bounds, and for
    x = 0 those raw-bound entries equal the oracle's t_d = 0 entries (whole periods reduce to the
    dead-time-free matrix, BASELINE north_star). The oracle itself reduces x_d = t_d mod t_r
    first, so this pins that reduction and its period bookkeeping against the physics."""
    rng = np.random.default_rng(300 + m)
    for k in (1, 2):
        f = random_flux(rng, 24, k, sigma_bins=(2, 8))
        d = f.t_r / f.n_bins
        for x in (0.0, float(rng.uniform(0.0, f.t_r)), float(rng.uniform(0.0, f.t_r))):
            if x > 0.0 and abs(x / d - round(x / d)) < 1e-6:
                continue          # keep a / Delta away from integers (the bin-edge tie, reading R4)
            td = m * f.t_r + x
            for i, j in [(int(i), j) for i in rng.integers(0, f.n_bins, 2) for j in range(f.n_bins)]:
                lam_j = oracle.lam(f, (j + 0.5) * d)
                I_raw = _raw_bound_integral(f, i, j, td)
                got = oracle.entry_eq4_unnorm(f, td, i, j)
                assert abs(-math.log(got / lam_j) - I_raw) <= 1e-8 * max(1.0, m * oracle.Lambda(f))
                if x == 0.0:
                    zero = oracle.entry_eq4_unnorm(f, 0.0, i, j)
                    assert abs(-math.log(zero / lam_j) - I_raw) <= 1e-8 * max(1.0, m * oracle.Lambda(f))
    # the raw bounds really sit m periods down the unrolled line (so the quadrature above never
    # saw a reduced dead time), and span less than one period plus one bin
    f = config(1).items[0].flux
    d = f.t_r / f.n_bins
    a = 3.5 * d + m * f.t_r + 75.0
    Da = (math.ceil(a / d) - 0.5) * d
    b = math.ceil((a - 5.5 * d) / f.t_r) * f.t_r + 5.5 * d
    assert m * f.t_r <= Da < b < Da + f.t_r + d


def test_p3b_decimal_whole_bins_land_on_a_bin_centre(oracle_lib):
    """t_d = k Delta written in decimal (Delta = 0.1 or 0.01, not binary fractions): the re-arm time
    s_i + t_d is exactly the bin centre s_{i+k}, reachable at zero distance, so the
    raw-bound integral (exact decimal rationals) is 0 for j = i + k and the entry is lambda(s_j)
    (E = 1). A shift rule that lets binary rounding push u = x_d / Delta above k moves that entry a
    whole period away (integral Lambda); reading R4 snaps u to k."""
    for t_r, N, tds in ((1.0, 10, ("0.3", "0.7", "1.3", "2.9")), (100.0, 10000, ("0.07", "1.13", "27.3"))):
        rng = np.random.default_rng(N)
        f = random_flux(rng, N, 1, t_r=t_r, sigma_bins=(2, 8))
        d = Fraction(str(t_r)) / N
        for td_s in tds:
            td = float(td_s)
            k = int(Fraction(td_s) / d) % N
            assert oracle.shift_l(f, td) == k
            for i in (0, 3, N // 2, N - 1):
                j = (i + k) % N
                a = (i + Fraction(1, 2)) * d + Fraction(td_s)
                s_j = (j + Fraction(1, 2)) * d
                Da = (math.ceil(a / d) - Fraction(1, 2)) * d
                b = math.ceil((a - s_j) / Fraction(str(t_r))) * Fraction(str(t_r)) + s_j
                assert b == Da                                   # zero distance, exactly
                got = oracle.entry_eq4_unnorm(f, td, i, j)
                assert got == oracle.lam(f, (j + 0.5) * (t_r / N)), (t_r, N, td_s, i)   # exp(-0) = 1


# -------------------------- P13 streamed x^T P~ (the only oracle route to pi P~ at N >= 16384)
@pytest.mark.parametrize("N,K,td_frac", [(97, 1, 0.37), (97, 2, 1.71), (256, 1, 2.42), (256, 2, 0.61)])
def test_p13_streamed_left_matvec(oracle_lib, N, K, td_frac):
    """oracle_left_matvec_streamed recomputes every row of Eq. 4 and accumulates x_i P~_i in long
    double over OpenMP threads. Pinned against numpy's matmul of the dense oracle matrix (a library
    product) for t_d below and above t_r, against single rows (x = e_i picks row i, so a transposed
    operand fails), and for thread-count independence."""
    rng = np.random.default_rng(1300 + N + K)
    f = random_flux(rng, N, K)
    td = td_frac * f.t_r
    P = oracle.build_eq4(f, td)
    Pl = P.astype(np.longdouble)           # the library product in extended precision, like the oracle's sum
    for x in (rng.uniform(0.0, 1.0, N), np.full(N, 1.0 / N)):
        y = oracle.left_matvec_streamed(f, td, x)
        want = (x.astype(np.longdouble) @ Pl).astype(np.float64)
        assert np.max(np.abs(y - want) / want) <= 2.3e-16
    for i in (0, N // 3, N - 1):
        e = np.zeros(N)
        e[i] = 1.0
        assert np.array_equal(oracle.left_matvec_streamed(f, td, e), P[i])
    X = rng.uniform(0.0, 1.0, (3, N))
    want = (X.astype(np.longdouble) @ Pl).astype(np.float64)
    assert np.max(np.abs(oracle.left_matvec_streamed_multi(f, td, X) - want) / want) <= 2.3e-16
    x = rng.uniform(0.0, 1.0, N)
    prev = oracle.max_threads()
    try:
        oracle.set_threads(1)
        y1 = oracle.left_matvec_streamed(f, td, x)
        oracle.set_threads(4)
        y4 = oracle.left_matvec_streamed(f, td, x)
    finally:
        oracle.set_threads(prev)
    assert np.max(np.abs(y1 - y4)) <= 1e-15 * max(1.0, float(np.max(np.abs(y1))))


# ------------------------------------------ P5 constant flux (S = 0): closed-form circulant chain
@pytest.mark.parametrize("B,N,td", [(1.0, 64, 37.3), (3.0, 50, 75.0), (10.0, 33, 250.0), (0.5, 16, 0.0)])
def test_p5_constant_flux_closed_form(oracle_lib, B, N, td):
    """With S = 0 the flux is B / t_r everywhere, so the integral of Eq. 4 is B/t_r times the
    distance from the re-arm bin centre to the next visit of s_j: P~_ij = r^d (1 - r) / (1 - r^N),
    r = exp(-B/N), d = (j - i - l) mod N; pi is uniform and |lambda_2| follows from the DFT of a
    circulant. Derived by hand from Eq. 3/4 for constant lambda (not from the oracle's code)."""
    f = Flux(100.0, N, (50.0,), (1.0,), (0.0,), B)
    P = oracle.build_eq4(f, td)
    x_d = math.fmod(td, 100.0)
    l = math.ceil(x_d / (100.0 / N) - 1e-9) % N    # the test's own shift: smallest bin offset >= x_d
    r = math.exp(-B / N)
    i = np.arange(N)[:, None]
    j = np.arange(N)[None, :]
    d = (j - i - l) % N
    expect = r ** d * (1.0 - r) / (1.0 - r ** N)
    assert np.max(np.abs(P - expect)) <= 1e-14
    pi = oracle.stationary_dense(P)
    assert np.max(np.abs(pi - 1.0 / N)) <= 1e-14
    # circulant eigenvalues: sum_d c_d w^{kd}; the second largest magnitude
    ev = np.abs(np.linalg.eigvals(P))
    ev.sort()
    k = np.arange(1, N)
    lam = (1 - r) / (1 - r * np.exp(2j * np.pi * k / N))
    assert abs(ev[-2] - np.max(np.abs(lam))) <= 1e-9


def test_p5_abs_lambda2_values(oracle_lib):
    """|lambda_2| of the S = 0 chain at N = 256: (1-r)/|1 - r e^{2 pi i/N}| for B = 1, 3, 10
    (0.15718, 0.43088, 0.84675 to 5 digits)."""
    N = 256
    for B, want in ((1.0, 0.15718), (3.0, 0.43088), (10.0, 0.84675)):
        f = Flux(100.0, N, (50.0,), (1.0,), (0.0,), B)
        ev = np.sort(np.abs(np.linalg.eigvals(oracle.build_eq4(f, 75.0))))
        assert abs(ev[-2] - want) < 5e-5


# ------------------------------------------- P6 structure of E_base (diag = 1, range)
def test_p6_exponent_structure(oracle_lib):
    rng = np.random.default_rng(5)
    for _ in range(3):
        f = random_flux(rng, 40, 2)
        Lam = oracle.Lambda(f)
        d = f.t_r / f.n_bins
        E = np.array([[oracle.entry_eq4_unnorm(f, 0.0, i, j) / oracle.lam(f, (j + 0.5) * d)
                       for j in range(f.n_bins)] for i in range(f.n_bins)])
        assert np.all(np.diag(E) == 1.0)                    # b = D(a) when j = i and t_d = 0
        assert np.all(E <= 1.0) and np.all(E >= math.exp(-Lam) * (1 - 1e-14))
        # along row i, E decays monotonically in the cyclic distance from s_i (the wrap term of
        # Eq. 5/6 sits below the diagonal): E_i,(i+d) is non-increasing in d = 0..N-1
        for i in range(f.n_bins):
            cyc = E[i, (i + np.arange(f.n_bins)) % f.n_bins]
            assert np.all(np.diff(cyc) <= 1e-15)
        # and the full-period product closes: E_i,i-1 = e^{-Lambda} * E_i-1... via one period
        assert abs(E[1, 0] - math.exp(-Lam) / E[0, 1]) <= 1e-13


# ------------------------------------------------------------ P7 solver agreement
@pytest.mark.parametrize("f,td", _rand_cases(3, 200, seed=11) + [(config(1).items[0].flux, 75.0)])
def test_p7_dense_vs_power(oracle_lib, f, td):
    P = oracle.build_eq4(f, td)
    pd = oracle.stationary_dense(P)
    pp, its, ch, ok = oracle.stationary_power(P, 1e-14)
    assert ok and ch < 1e-14
    assert np.sum(np.abs(pd - pp)) <= 1e-13
    assert abs(pd.sum() - 1.0) <= 1e-14 and np.all(pd > 0)
    assert np.sum(np.abs(pd @ P - pd)) <= 1e-14


# ------------------------------------------------------------ P8 tiny analytic chains
def test_p8_two_state(oracle_lib):
    P = np.array([[0.9, 0.1], [0.2, 0.8]])
    want = np.array([2.0 / 3.0, 1.0 / 3.0])
    assert np.max(np.abs(oracle.stationary_dense(P) - want)) <= 1e-15
    pp, its, ch, ok = oracle.stationary_power(P, 1e-15)
    assert ok and np.max(np.abs(pp - want)) <= 1e-14


def _exact_stationary(Pq):
    """pi (P - I) = 0, sum pi = 1, in exact rationals (Gauss-Jordan)."""
    n = len(Pq)
    A = [[Pq[c][r] - (1 if r == c else 0) for c in range(n)] for r in range(n)]
    b = [Fraction(0)] * n
    A[-1] = [Fraction(1)] * n
    b[-1] = Fraction(1)
    for k in range(n):
        p = next(r for r in range(k, n) if A[r][k] != 0)
        A[k], A[p], b[k], b[p] = A[p], A[k], b[p], b[k]
        for r in range(n):
            if r != k and A[r][k] != 0:
                m = A[r][k] / A[k][k]
                A[r] = [x - m * y for x, y in zip(A[r], A[k])]
                b[r] -= m * b[k]
    return [b[k] / A[k][k] for k in range(n)]


@pytest.mark.parametrize("N", [2, 3, 5])
def test_p8_brute_force_rational(oracle_lib, N):
    rng = np.random.default_rng(N)
    f = random_flux(rng, N, 1)
    P = oracle.build_eq4(f, float(rng.uniform(0, 150)))
    Pq = [[Fraction(x) for x in row] for row in P]
    # renormalise exactly so the rational chain is exactly stochastic
    Pq = [[x / sum(row) for x in row] for row in Pq]
    exact = np.array([float(x) for x in _exact_stationary(Pq)])
    assert np.max(np.abs(oracle.stationary_dense(P) - exact)) <= 1e-15
    pp, _, _, ok = oracle.stationary_power(P, 1e-15)
    assert ok and np.max(np.abs(pp - exact)) <= 1e-14


# ----------------------------- P9 / P12: the integral of Eq. 3/4 by quadrature (Thm 1)
def _lam_tilde_integral(f, lo, hi):
    """int_lo^hi lambda~ by adaptive quadrature of the oracle's pointwise lambda, split at period
    boundaries and at the pulse centres (independent of the closed-form F)."""
    total = 0.0
    k0 = math.floor(lo / f.t_r)
    k1 = math.floor(hi / f.t_r)
    for k in range(k0, k1 + 1):
        a = max(lo, k * f.t_r) - k * f.t_r
        b = min(hi, (k + 1) * f.t_r) - k * f.t_r
        if b <= a:
            continue
        pts = [p for p in f.tau if a < p < b]
        v, _ = integrate.quad(lambda t: oracle.lam(f, t), a, b, points=pts or None, limit=400,
                              epsabs=1e-13, epsrel=1e-12)
        total += v
    return total


def test_p12_F_vs_quadrature(oracle_lib):
    rng = np.random.default_rng(12)
    for _ in range(5):
        f = random_flux(rng, 100, 2)
        for t in rng.uniform(0, f.t_r, 4):
            assert abs(oracle.F(f, t) - _lam_tilde_integral(f, 0.0, t)) <= 1e-9 * max(1.0, oracle.Lambda(f))
        # Lambda = S + B when the pulses sit well inside the period (reading R5)
    f = config(1).items[0].flux
    assert abs(oracle.Lambda(f) - 0.6) <= 1e-15


def test_p9_theorem1_continuous(oracle_lib):
    """Theorem 1 in continuous variables (Remark 1): with a = x_k + x_d and
    b = ceil((a - x_{k+1}) / t_r) t_r + x_{k+1}, int_a^b lambda~ equals
    Lambda 1{x_k' > x_{k+1}} + F(x_{k+1}) - F(x_k'), x_k' = (x_k + x_d) mod t_r.
    The left side is quadrature; the right side uses the oracle's closed-form F."""
    rng = np.random.default_rng(9)
    f = random_flux(rng, 100, 1, sigma_bins=(5, 20))
    Lam = oracle.Lambda(f)
    for _ in range(60):
        xk, xk1 = rng.uniform(0, f.t_r, 2)
        td = rng.uniform(0, 3 * f.t_r)
        xd = math.fmod(td, f.t_r)
        a = xk + xd
        b = math.ceil((a - xk1) / f.t_r) * f.t_r + xk1
        lhs = _lam_tilde_integral(f, a, b)
        xkp = math.fmod(xk + xd, f.t_r)
        rhs = Lam * (xkp > xk1) + oracle.F(f, xk1) - oracle.F(f, xkp)
        assert abs(lhs - rhs) <= 1e-8 * max(1.0, Lam)


def test_p9_discrete_entries_are_integrals(oracle_lib):
    """Each unnormalised oracle entry is lambda(s_j) exp(-int_{D(a)}^{D(b)} lambda~): recover the
    integral and compare with quadrature between the bin-centre limits."""
    rng = np.random.default_rng(19)
    f = random_flux(rng, 24, 2, sigma_bins=(2, 8))
    d = f.t_r / f.n_bins
    for _ in range(40):
        i, j = (int(x) for x in rng.integers(0, f.n_bins, 2))
        td = float(rng.uniform(0, 2.5 * f.t_r))
        x_d = math.fmod(td, f.t_r)
        a = (i + 0.5) * d + x_d
        Da = (math.ceil(a / d) - 0.5) * d
        b = math.ceil((a - (j + 0.5) * d) / f.t_r) * f.t_r + (j + 0.5) * d
        I = -math.log(oracle.entry_eq4_unnorm(f, td, i, j) / oracle.lam(f, (j + 0.5) * d))
        assert abs(I - _lam_tilde_integral(f, Da, b)) <= 1e-8


# ------------------------------------------------- P4 vanishing flux (t_d = 0 i.i.d. limit)
def test_p4_vanishing_flux(oracle_lib):
    """As S, B -> 0 every E_ij -> 1, so every row -> lambda / sum(lambda) and pi -> lambda/sum(lambda)
    at any dead time, with an O(eps) error: L1/eps must be constant over decades of eps."""
    base = config(1).items[0].flux
    d = base.t_r / base.n_bins
    ratios = []
    for eps in (1e-2, 1e-3, 1e-4, 1e-5):
        f = base.scaled(eps)
        lam = np.array([oracle.lam(f, (j + 0.5) * d) for j in range(f.n_bins)])
        pi = oracle.stationary_dense(oracle.build_eq4(f, 75.0))
        ratios.append(np.sum(np.abs(pi - lam / lam.sum())) / eps)
    assert ratios[-1] > 0
    assert abs(ratios[2] / ratios[3] - 1) < 1e-3 and abs(ratios[1] / ratios[3] - 1) < 1e-2
    assert 0.13 < ratios[-1] < 0.15      # SURVEY P4 scratch: c = 0.1384 for this shape


# ---------------------------------------------------- P11 structured O(N) cross-check (F3)
def test_p11_structured_matvec(oracle_lib):
    """Independent O(N) algorithm: with w_j = lambda_j e^{-F_j} and D_r = sum_{j>=r} w_j +
    e^{-Lambda} sum_{j<r} w_j, x^T P~0 = w * (cumsum(x/D) + e^{-Lambda} (sum - cumsum)(x/D))
    (rank-1 semiseparable form of E_base). Built here from the oracle's pointwise
    lambda and F only, then compared with the oracle's Eq. 4 matrix and its pi."""
    f = config(2).items[3].flux.with_bins(512)
    td = 50.0
    N = f.n_bins
    d = f.t_r / N
    s = (np.arange(N) + 0.5) * d
    lam = np.array([oracle.lam(f, t) for t in s])
    Fv = np.array([oracle.F(f, t) for t in s])
    Lam = oracle.Lambda(f)
    w = lam * np.exp(-Fv)
    U = np.cumsum(w[::-1])[::-1]
    L = np.concatenate([[0.0], np.cumsum(w)[:-1]])
    D = U + math.exp(-Lam) * L
    l = oracle.shift_l(f, td)

    def step(pi):
        x = np.roll(pi, l)               # x_r = pi[(r - l) mod N]
        z = x / D
        c = np.cumsum(z)
        y = w * (c + math.exp(-Lam) * (c[-1] - c))
        return y / y.sum()

    pi = np.full(N, 1.0 / N)
    for _ in range(500):
        nxt = step(pi)
        if np.sum(np.abs(nxt - pi)) < 1e-15:
            pi = nxt
            break
        pi = nxt
    P = oracle.build_eq4(f, td)
    x = np.random.default_rng(0).random(N)
    x /= x.sum()
    y_dense = x @ P
    y_struct = step(x) * np.sum(x @ P)
    assert np.max(np.abs(y_dense - y_struct)) <= 1e-15
    assert np.sum(np.abs(oracle.stationary_dense(P) - pi)) <= 1e-13


# ------------------------------------------------------------ P10 Monte Carlo
def _bin_integrated_fa(f, n_hist):
    edges = np.linspace(0.0, f.t_r, n_hist + 1)
    Fe = np.array([oracle.F(f, e) for e in edges])
    return np.diff(Fe) / Fe[-1]


def _mc_freq(f, td, seed, n_hist, n_batches=20, per_batch=50000):
    h = oracle.monte_carlo(f, td, seed, 1000, per_batch, n_batches, n_hist)
    fr = h / per_batch
    return fr.mean(axis=0), fr.std(axis=0, ddof=1) / math.sqrt(n_batches)


def test_p10_mc_sampler_no_deadtime(oracle_lib):
    """t_d = 0: registrations are i.i.d. f_a, so the MC histogram is the bin-integrated f_a."""
    f = Flux(100.0, 16, (40.0,), (5.0,), (2.0,), 1.0)
    m, se = _mc_freq(f, 0.0, 1, 16)
    assert np.all(np.abs(m - _bin_integrated_fa(f, 16)) <= 4.5 * se + 1e-12)


def test_p10_mc_constant_flux_uniform(oracle_lib):
    f = Flux(100.0, 16, (40.0,), (5.0,), (0.0,), 2.0)
    m, se = _mc_freq(f, 75.0, 2, 16)
    assert np.all(np.abs(m - 1.0 / 16) <= 4.5 * se)


def test_p10_mc_timestamps_dead_time_and_renewal(oracle_lib):
    """One chain's registrations (the stream the GPU Monte Carlo is replayed against): offsets in
    [0, t_r), absolute times T = q t_r + t strictly increasing with every gap >= t_d (the SPAD is dead
    for t_d after each registration), and at constant flux (S = 0, rate B / t_r) the gaps are
    t_d + Exp(B / t_r): mean t_d + t_r / B and variance (t_r / B)^2 within 5 standard errors (renewal
    process)."""
    f = Flux(100.0, 16, (40.0,), (5.0,), (0.0,), 2.0)
    td = 37.5
    q, t = oracle.mc_timestamps(f, td, 99, 200000)
    assert np.all((t >= 0.0) & (t < f.t_r))
    T = q.astype(np.float64) * f.t_r + t
    gaps = np.diff(T)
    assert np.all(gaps >= td * (1 - 1e-12))
    mean_exp, n = f.t_r / f.background, gaps.size
    assert abs(gaps.mean() - (td + mean_exp)) <= 5 * mean_exp / math.sqrt(n)
    assert abs(gaps.var() - mean_exp ** 2) <= 5 * mean_exp ** 2 * math.sqrt(8.0 / n)   # Var(X^2) = 8 m^4 - m^4
    g = config(1).items[0].flux                         # a pulsed flux: the gating holds there too
    q, t = oracle.mc_timestamps(g, 75.0, 7, 20000)
    assert np.all(np.diff(q.astype(np.float64) * g.t_r + t) >= 75.0 * (1 - 1e-12))


def test_p14_left_matvec(oracle_lib):
    """oracle.left_matvec (the product inside stationary_power and the CPU baseline's timing) equals
    the extended-precision library product x @ rows, and e_i picks row i."""
    rng = np.random.default_rng(14)
    rows = rng.uniform(0.0, 1.0, (300, 77))
    x = rng.uniform(0.0, 1.0, 300)
    want = (x.astype(np.longdouble) @ rows.astype(np.longdouble)).astype(np.float64)
    assert np.max(np.abs(oracle.left_matvec(rows, x) - want) / want) <= 2.3e-16
    e = np.zeros(300)
    e[123] = 1.0
    assert np.array_equal(oracle.left_matvec(rows, e), rows[123])


@pytest.mark.parametrize("td", [75.0, 130.0])
def test_p10_mc_vs_chain(oracle_lib, td):
    """The chain's pi (fine N, aggregated to 16 comparison bins) against the continuous-time MC
    of P:60: every bin within 4 SE (batch means) + 2 |pi_N - pi_2N| (first-order discretisation
    bias)."""
    f = Flux(100.0, 512, (40.0,), (5.0,), (2.0,), 1.0)
    m, se = _mc_freq(f, td, 3, 16)
    aggs = []
    for n in (512, 1024):
        P = oracle.build_eq4(f.with_bins(n), td)
        pi, _, _, ok = oracle.stationary_power(P, 1e-14)
        assert ok
        aggs.append(pi.reshape(16, -1).sum(axis=1))
    bias = np.abs(aggs[0] - aggs[1])
    assert np.all(np.abs(m - aggs[1]) <= 4.0 * se + 2.0 * bias)
    # and the dead-time distortion is real: the MC is far from the undistorted f_a
    assert np.max(np.abs(m - _bin_integrated_fa(f, 16))) > 20 * np.max(se)


# ------------------------------------------------------------ regression fixture (not a pin)
def test_golden_config1_regression(oracle_lib):
    import json
    import os
    g = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "config1_oracle.json")))
    it = config(1).items[0]
    P = oracle.build_eq4(it.flux, it.t_d)
    for r, row in g["rows"].items():
        assert np.max(np.abs(P[int(r)] - np.array(row))) <= 1e-15
    assert np.sum(np.abs(oracle.stationary_dense(P) - np.array(g["pi"]))) <= 1e-14


# ===================================================== f1: spectral analysis (§4)
# Pins of oracle.second_eigenvalue / mixing_steps / bin_trajectory against closed forms derived by
# hand (two-state chain, a rotation-plus-teleport 3-state chain with a complex pair, the S = 0
# circulant with its DFT spectrum incl. the phase the shift l adds), and against the dynamics they
# describe (decay rate and oscillation of a trajectory on a model chain).

@pytest.mark.parametrize("a,b", [(0.1, 0.2), (0.3, 0.45), (0.7, 0.9), (0.05, 0.95)])
def test_f1_two_state_lambda2(a, b):
    """[[1-a, a], [b, 1-b]]: eigenvalues 1 and 1 - a - b; phase 0 if positive, pi if negative."""
    P = np.array([[1 - a, a], [b, 1 - b]])
    lam = oracle.second_eigenvalue(P)
    assert abs(lam - (1 - a - b)) <= 1e-14
    ph = math.atan2(lam.imag, lam.real)
    assert abs(ph - (0.0 if 1 - a - b >= 0 else math.pi)) <= 1e-14


@pytest.mark.parametrize("alpha", [0.3, 0.8, 0.95])
def test_f1_rotation_chain_complex_pair(alpha):
    """P = alpha Cyc + (1 - alpha) J / 3 (Cyc the cyclic shift, J all ones): Cyc has eigenvalues
    1, w, w^2 (w = e^{2 pi i / 3}) on eigenvectors orthogonal to 1 except the first, and J kills
    those, so lambda_2 = alpha e^{2 pi i / 3}: modulus alpha, phase 2 pi / 3."""
    Cyc = np.roll(np.eye(3), 1, axis=1)
    P = alpha * Cyc + (1 - alpha) * np.ones((3, 3)) / 3
    lam = oracle.second_eigenvalue(P)
    assert abs(abs(lam) - alpha) <= 1e-13
    assert abs(math.atan2(lam.imag, lam.real) - 2 * math.pi / 3) <= 1e-13


@pytest.mark.parametrize("B,N,td", [(1.0, 64, 37.3), (3.0, 50, 75.0), (10.0, 33, 250.0), (0.5, 128, 10.0)])
def test_f1_circulant_lambda2_with_phase(oracle_lib, B, N, td):
    """S = 0: P~ is circulant with first-row entries a_m = c r^{(m - l) mod N} (pin P5), so its
    eigenvalues are mu_k = sum_m a_m w^{mk} = w^{lk} (1 - r) / (1 - r w^k), w = e^{2 pi i / N}.
    The modulus is largest at k = 1, N - 1 (a conjugate pair); its phase carries the shift l."""
    f = Flux(100.0, N, (50.0,), (1.0,), (0.0,), B)
    P = oracle.build_eq4(f, td)
    l = math.ceil(math.fmod(td, 100.0) / (100.0 / N) - 1e-9) % N
    r = math.exp(-B / N)
    w = np.exp(2j * np.pi / N)
    mu = w ** (l * 1) * (1 - r) / (1 - r * w)
    want = complex(mu.real, abs(mu.imag))
    lam = oracle.second_eigenvalue(P)
    assert abs(abs(lam) - abs(mu)) <= 1e-12
    assert abs(lam - want) <= 1e-10


def test_f1_brute_force_char_poly():
    """n = 8 random positive stochastic matrix: the characteristic polynomial in exact rationals
    (Faddeev-LeVerrier) vanishes at the oracle's lambda_2, and no root of it other than 1 has a
    larger modulus (roots located by the argument principle on a circle through |lambda_2|)."""
    rng = np.random.default_rng(8)
    n = 8
    Q = [[Fraction(int(rng.integers(1, 50))) for _ in range(n)] for _ in range(n)]
    for row in Q:
        s = sum(row)
        row[:] = [x / s for x in row]
    P = np.array([[float(x) for x in row] for row in Q])
    # Faddeev-LeVerrier: c_n = 1, M_k = A M_{k-1} + c_{n-k+1} I, c_{n-k} = -tr(A M_k) / k
    I = [[Fraction(int(i == j)) for j in range(n)] for i in range(n)]
    def mul(X, Y):
        return [[sum(X[i][k] * Y[k][j] for k in range(n)) for j in range(n)] for i in range(n)]
    c = [Fraction(0)] * (n + 1)
    c[n] = Fraction(1)
    Mk = [[Fraction(0)] * n for _ in range(n)]
    for k in range(1, n + 1):
        Mk = mul(Q, Mk)
        for i in range(n):
            Mk[i][i] += c[n - k + 1]
        AM = mul(Q, Mk)
        c[n - k] = -sum(AM[i][i] for i in range(n)) / k
    coef = [float(x) for x in c]                        # ascending powers
    def poly(z):
        return sum(cf * z ** p for p, cf in enumerate(coef))
    assert abs(poly(1.0)) <= 1e-12                      # stochastic: 1 is a root
    lam = oracle.second_eigenvalue(P)
    assert abs(poly(lam)) <= 1e-10
    # number of roots inside |z| < rho by the argument principle (numerical winding number)
    def n_roots_inside(rho):
        t = np.linspace(0, 2 * np.pi, 20001)
        z = rho * np.exp(1j * t)
        v = np.array([poly(x) for x in z])
        return int(round(np.sum(np.diff(np.unwrap(np.angle(v)))) / (2 * np.pi)))
    rho = abs(lam)
    mult = 2 if abs(lam.imag) > 1e-12 else 1
    assert n_roots_inside(rho * (1 + 1e-6)) - n_roots_inside(rho * (1 - 1e-6)) == mult
    assert n_roots_inside(min(0.999999, rho * (1 + 1e-6))) == n - 1   # only the Perron root is outside


def test_f1_mixing_closed_forms():
    """Rank-1 chain (every row = pi) mixes in one step. Two-state chain: e_i P^n - pi =
    lambda^n (e_i - pi), so TV_i(n) = |lambda|^n (1 - pi_i) and n = ceil(log(eps / max_i(1 - pi_i)) /
    log|lambda|)."""
    pi = np.array([0.2, 0.5, 0.3])
    n, first = oracle.mixing_steps(np.tile(pi, (3, 1)), pi, 1e-3)
    assert n == 1 and np.all(first == 1)
    for a, b, eps in ((0.1, 0.2, 1e-3), (0.6, 0.9, 1e-4), (0.05, 0.05, 1e-3)):
        P = np.array([[1 - a, a], [b, 1 - b]])
        p = np.array([b / (a + b), a / (a + b)])
        lam = abs(1 - a - b)
        want = math.ceil(math.log(eps / np.max(1 - p)) / math.log(lam))
        n, first = oracle.mixing_steps(P, p, eps)
        assert n == want
        assert list(first) == [math.ceil(math.log(eps / (1 - p[i])) / math.log(lam)) for i in range(2)]


def test_f1_mixing_circulant_symmetry_and_background_trend(oracle_lib):
    """S = 0: every start mixes in the same number of steps (circulant symmetry). Paper §4.1:
    mixing slows as B grows ("gap decreases as background B increases"): non-decreasing over
    B in {0.1, 3, 6, 9} at fixed S."""
    f = Flux(100.0, 64, (50.0,), (1.0,), (0.0,), 3.0)
    P = oracle.build_eq4(f, 75.0)
    n, first = oracle.mixing_steps(P, np.full(64, 1 / 64), 1e-3)
    assert np.all(first == n)
    steps = []
    for B in (0.1, 3.0, 6.0, 9.0):
        g = Flux(100.0, 128, (40.0,), (1.0,), (2.0,), B)
        P = oracle.build_eq4(g, 75.0)
        steps.append(oracle.mixing_steps(P, oracle.stationary_dense(P), 1e-3)[0])
    assert steps == sorted(steps)


def test_f1_trajectory_closed_forms():
    """start = pi stays at pi[bin]; two-state chain from e_1: pi_1 + (1 - pi_1) lambda^n."""
    a, b = 0.3, 0.5
    P = np.array([[1 - a, a], [b, 1 - b]])
    p = np.array([b / (a + b), a / (a + b)])
    tr, _ = oracle.bin_trajectory(P, p, 0, 20)
    assert np.max(np.abs(tr - p[0])) <= 1e-15
    tr, _ = oracle.bin_trajectory(P, np.array([1.0, 0.0]), 0, 30)
    n = np.arange(31)
    assert np.max(np.abs(tr - (p[0] + (1 - p[0]) * (1 - a - b) ** n))) <= 1e-15


@pytest.mark.parametrize("S,B,td", [(2.0, 3.0, 75.0), (1.0, 6.0, 75.0), (1.0, 9.0, 95.0)])
def test_f1_trajectory_decay_matches_lambda2(oracle_lib, S, B, td):
    """Fig. 4 caption: amplitude decays at |lambda_2| per step and oscillates with
    arg(lambda_2). Checked on a model chain: the residual r_n = traj_n - pi[bin] from a point start
    fits r_n ~ Re(c lambda_2^n) over the tail (least squares in (Re c, Im c) with the oracle's
    lambda_2) to 1e-4 relative over 30 steps once the third mode has decayed, while the same fit with
    |lambda_2| perturbed by 2% fails."""
    f = Flux(100.0, 96, (40.0,), (0.8,), (S,), B)
    P = oracle.build_eq4(f, td)
    pi = oracle.stationary_dense(P)
    lam = oracle.second_eigenvalue(P)
    start = np.zeros(96)
    start[5] = 1.0
    mods = np.sort(np.abs(np.linalg.eigvals(P)))[::-1]
    third = mods[3] if abs(mods[1] - mods[2]) < 1e-9 else mods[2]   # next mode after the pair / real root
    n0 = int(math.ceil(math.log(1e-5) / math.log(third / abs(lam))))
    n1 = n0 + 30
    bin_ = int(np.argmax(pi))
    tr, _ = oracle.bin_trajectory(P, start, bin_, n1)
    r = tr[n0:n1 + 1] - pi[bin_]
    n = np.arange(n0, n1 + 1)

    def fit_err(lm):
        A = np.stack([(lm ** n).real, -(lm ** n).imag], axis=1) if abs(lm.imag) > 0 else (lm.real ** n)[:, None]
        coef, *_ = np.linalg.lstsq(A, r, rcond=None)
        return np.max(np.abs(A @ coef - r)) / np.max(np.abs(r))
    good, bad = fit_err(lam), fit_err(lam * 1.02)
    assert good <= 1e-4 and bad > 1e-3 and bad > 30 * good, (good, bad)
