"""Monte Carlo of the detection process on the GPU (pytest -m gpu).

Both sides implement the same counter-based generator (splitmix64, one draw per registration from
the chain seed), so a GPU chain is replayed draw for draw by the CPU oracle (oracle.mc_timestamps):
the registration times must agree up to the two root finders' tolerances. The histograms are then
checked exactly against the recorded timestamps, and statistically against what the paper and the
oracle fix: the chain's pi (the MC is the model's ground truth), the uniform law at S = 0 and
the bin-integrated f_a at t_d = 0."""
import math

import numpy as np
import pytest
import torch

import oracle
from workloads import Flux, config

pytestmark = pytest.mark.gpu

GAMMA = 0xD1B54A32D192ED03


@pytest.fixture(scope="module")
def spl():
    assert torch.cuda.is_available(), "GPU tests need a B200"
    from paper_2509_20500_b200 import build
    build.build()
    import paper_2509_20500_b200 as s
    return s


def _np(t):
    return t.detach().cpu().numpy()


def _seed(seed, c):
    return (seed + c * GAMMA) % 2 ** 64


def _items_of(flux):
    tot = float(sum(flux.signal))
    shape = Flux(flux.t_r, flux.n_bins, flux.tau, flux.sigma, tuple(s / tot for s in flux.signal), 1.0)
    return shape, tot


REPLAY = [(config(1).items[0].flux, 75.0), (Flux(100.0, 64, (30.0, 70.0), (2.0, 4.0), (1.5, 0.7), 0.6), 130.0),
          (Flux(200.0, 64, (60.0,), (1.0,), (0.3,), 2.0), 430.0)]


@pytest.mark.parametrize("f,td", REPLAY, ids=["config1", "two-pulse", "td>t_r"])
def test_mc_chains_replay_on_oracle(spl, f, td):
    """Chains of two items (S and B differ) x 64 runs, first 300 registrations recorded; chains 0, 17,
    63 of each item replayed by the oracle from the same seed: equal periods, offsets within 1e-9 t_r."""
    shape, tot = _items_of(f)
    S = [tot, 0.5 * tot]
    B = [f.background, 2.0 * f.background]
    n_runs, n_rec, seed = 64, 300, 12345
    hist, q, t = spl.monte_carlo(shape, S, B, [td, td], seed, n_runs, 32, n_burn=0, n_regs=n_rec, n_record=n_rec)
    q, t = _np(q), _np(t)
    for m in range(2):
        fm = Flux(f.t_r, f.n_bins, f.tau, f.sigma, tuple(S[m] * np.array(shape.signal)), B[m])
        for run in (0, 17, 63):
            c = m * n_runs + run
            qo, to = oracle.mc_timestamps(fm, td, _seed(seed, c), n_rec)
            T_gpu = q[c] * f.t_r + t[c]
            T_or = qo * f.t_r + to
            assert np.max(np.abs(T_gpu - T_or)) <= 1e-9 * f.t_r, (m, run)


def test_mc_histogram_matches_recorded_timestamps(spl):
    """Binning, burn-in and the stop rule, exactly: the histogram of every run equals the host binning
    of its recorded timestamps k in [n_burn, n_burn + n_regs)."""
    f = config(1).items[0].flux
    shape, tot = _items_of(f)
    n_burn, n_regs, n_hist = 50, 400, 40
    hist, q, t = spl.monte_carlo(shape, [tot], [f.background], [75.0], 7, 96, n_hist, n_burn=n_burn,
                                 n_regs=n_regs, n_record=n_burn + n_regs)
    t = _np(t)[:, n_burn:]
    dh = f.t_r / n_hist
    b = np.ceil(t / dh).astype(np.int64) - 1
    b[b < 0] = n_hist - 1
    b[b >= n_hist] = n_hist - 1
    want = np.stack([np.bincount(r, minlength=n_hist) for r in b])
    assert np.array_equal(_np(hist[0]), want)


def test_mc_cycles_mode(spl):
    """n_cycles: counted registrations are exactly those in the first n_cycles periods after burn-in."""
    f = config(1).items[0].flux
    shape, tot = _items_of(f)
    hist, q, t = spl.monte_carlo(shape, [tot], [f.background], [75.0], 9, 32, 16, n_burn=0, n_cycles=60,
                                 n_record=400)
    q = _np(q)
    counts = _np(hist[0]).sum(axis=1)
    # the run stops at (and records) its first registration at or beyond period 60; slots after it
    # are never written
    stop = np.array([int(np.argmax(r >= 60)) for r in q])
    assert np.all(q[np.arange(q.shape[0]), stop] >= 60)
    assert all(np.all(np.diff(r[:s + 1]) >= 0) for r, s in zip(q, stop))
    assert np.array_equal(counts, stop)


def _freq(h):
    """Per-run frequencies [runs, bins] -> mean and standard error over runs."""
    fr = h / h.sum(axis=1, keepdims=True)
    return fr.mean(axis=0), fr.std(axis=0, ddof=1) / math.sqrt(fr.shape[0])


def _bin_integrated_fa(f, n):
    edges = np.linspace(0.0, f.t_r, n + 1)
    Fe = np.array([oracle.F(f, e) for e in edges])
    return np.diff(Fe) / Fe[-1]


@pytest.mark.parametrize("td", [75.0, 130.0])
def test_mc_vs_chain_pi(spl, td):
    """The chain's pi at fine N (aggregated to 16 comparison bins) within 4 SE (over 512 independent
    runs of 20000 registrations) + 2 |pi_N - pi_2N| of the GPU MC; the dead-time distortion from f_a
    is resolved far beyond the noise."""
    f = Flux(100.0, 512, (40.0,), (5.0,), (2.0,), 1.0)
    shape, tot = _items_of(f)
    h = _np(spl.monte_carlo(shape, [tot], [f.background], [td], 2024, 512, 16, n_burn=200, n_regs=20000)[0])
    m, se = _freq(h)
    aggs = []
    for n in (512, 1024):
        P = oracle.build_eq4(f.with_bins(n), td)
        aggs.append(oracle.stationary_dense(P).reshape(16, -1).sum(axis=1))
    bias = np.abs(aggs[0] - aggs[1])
    assert np.all(np.abs(m - aggs[1]) <= 4.0 * se + 2.0 * bias)
    assert np.max(np.abs(m - _bin_integrated_fa(f, 16))) > 20 * np.max(se)


def test_mc_special_cases(spl):
    """S = 0: uniform timestamps; t_d = 0: i.i.d. f_a, the bin-integrated arrival pdf."""
    f0 = Flux(100.0, 16, (40.0,), (5.0,), (1.0,), 2.0)
    h = _np(spl.monte_carlo(f0, [0.0], [2.0], [75.0], 5, 256, 16, n_burn=100, n_regs=5000)[0])
    m, se = _freq(h)
    assert np.all(np.abs(m - 1.0 / 16) <= 4.5 * se)
    f = Flux(100.0, 16, (40.0,), (5.0,), (2.0,), 1.0)
    shape, tot = _items_of(f)
    h = _np(spl.monte_carlo(shape, [tot], [1.0], [0.0], 6, 256, 16, n_burn=100, n_regs=5000)[0])
    m, se = _freq(h)
    assert np.all(np.abs(m - _bin_integrated_fa(f, 16)) <= 4.5 * se + 1e-12)


def test_mc_rejects(spl):
    f = config(1).items[0].flux
    with pytest.raises(spl.SplidarError):
        spl.monte_carlo(f, [1.0], [0.1], [75.0], 1, 0, 16, n_regs=10)        # no runs
    with pytest.raises(spl.SplidarError):
        spl.monte_carlo(f, [1.0], [0.1], [75.0], 1, 4, 16)                   # neither n_regs nor n_cycles
    with pytest.raises(spl.SplidarError):
        spl.monte_carlo(f, [1.0], [0.1], [-1.0], 1, 4, 16, n_regs=10)        # negative dead time


def test_mc_split_subchains(spl):
    """n_split = 4: chain c = (m * n_runs + run) * 4 + sub is replayed by the oracle from its own seed,
    and run r's histogram is exactly the binning of its 4 sub-chains' counted registrations."""
    f = Flux(100.0, 64, (30.0, 70.0), (2.0, 4.0), (1.5, 0.7), 0.6)
    shape, tot = _items_of(f)
    n_runs, n_split, n_burn, n_regs, n_hist, seed = 8, 4, 20, 400, 24, 99
    hist, q, t = spl.monte_carlo(shape, [tot], [f.background], [57.0], seed, n_runs, n_hist, n_burn=n_burn,
                                 n_regs=n_regs, n_record=n_burn + n_regs // n_split, n_split=n_split)
    q, t = _np(q), _np(t)
    assert q.shape[0] == n_runs * n_split
    c = 1 * n_split + 2
    qo, to = oracle.mc_timestamps(f, 57.0, _seed(seed, c), n_burn + n_regs // n_split)
    assert np.max(np.abs((q[c] * f.t_r + t[c]) - (qo * f.t_r + to))) <= 1e-9 * f.t_r
    dh = f.t_r / n_hist
    for run in range(n_runs):
        tt = t[run * n_split:(run + 1) * n_split, n_burn:].ravel()
        b = np.ceil(tt / dh).astype(np.int64) - 1
        b[b < 0] = n_hist - 1
        b[b >= n_hist] = n_hist - 1
        assert np.array_equal(_np(hist[0, run]), np.bincount(b, minlength=n_hist))
    with pytest.raises(spl.SplidarError):    # budget not divisible by n_split
        spl.monte_carlo(shape, [tot], [f.background], [57.0], seed, 2, 8, n_regs=401, n_split=4)
