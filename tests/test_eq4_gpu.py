"""the element-wise Eq. 4 construction on the GPU (pytest -m gpu), against the
CPU oracle's Eq. 4 (same definition) and against Theorem 2's construction on the GPU
(build_base + the row permutation), which it must reproduce up to rounding."""
import numpy as np
import pytest
import torch

import oracle
from workloads import config, parity_cases

from ._structured import sampled_rows

pytestmark = pytest.mark.gpu

CASES = parity_cases()
IDS = [f"N{c.flux.n_bins}-K{c.flux.n_pulses}-td{c.t_d:.2f}" for c in CASES]


@pytest.fixture(scope="module")
def spl():
    assert torch.cuda.is_available(), "GPU tests need a B200"
    from paper_2509_20500_b200 import build
    build.build()
    import paper_2509_20500_b200 as s
    return s


def _np(t):
    return t.detach().cpu().numpy()


@pytest.mark.parametrize("case", CASES, ids=IDS)
def test_eq4_vs_oracle_f64(spl, case):
    f = case.flux
    got = _np(spl.build_eq4(f, case.t_d))
    want = oracle.build_eq4(f, case.t_d)
    assert np.max(np.abs(got - want)) <= 1e-12
    assert np.max(np.abs(got.sum(axis=1) - 1.0)) <= 1e-12


@pytest.mark.parametrize("case", CASES[::3], ids=IDS[::3])
def test_eq4_vs_oracle_f32(spl, case):
    f = case.flux
    got = _np(spl.build_eq4(f, case.t_d, torch.float32)).astype(np.float64)
    assert np.max(np.abs(got - oracle.build_eq4(f, case.t_d))) <= 1e-5


@pytest.mark.parametrize("case", CASES[::2], ids=IDS[::2])
def test_eq4_equals_theorem2(spl, case):
    """Eq. 4 element by element == J_l P~0 from the reparameterised base matrix (Thm 2)."""
    f = case.flux
    P0 = spl.build_base(f)
    P = spl.apply_deadtime(P0, f.t_r, case.t_d)
    assert torch.max(torch.abs(spl.build_eq4(f, case.t_d) - P)).item() <= 1e-13


@pytest.mark.parametrize("k", [3, 5])
def test_eq4_large_sampled_rows(spl, k):
    """Configs 3 and 5 (N = 4096, 32768): sampled rows against the oracle's Eq. 4 rows, and the whole
    matrix against Theorem 2's construction on the device."""
    it = config(k).items[0]
    f = it.flux
    P = spl.build_eq4(f, it.t_d)
    N = f.n_bins
    rows = sorted({0, 1, N - 1, 777 % N, N // 2, N // 3})
    want = sampled_rows(f, it.t_d, rows)
    got = np.stack([_np(P[r]) for r in rows])
    assert np.max(np.abs(got - want)) <= 1e-12
    P0 = spl.build_base(f)
    l = spl.shift(f.t_r, N, it.t_d)
    err = 0.0
    for r0 in range(0, N, 4096):   # row blocks: J_l P~0 without materialising a second matrix
        r1 = min(N, r0 + 4096)
        src = (torch.arange(r0, r1, device="cuda") + l) % N
        err = max(err, torch.max(torch.abs(P[r0:r1] - P0[src])).item())
    assert err <= 1e-13
    del P, P0
    torch.cuda.empty_cache()


def test_eq4_rejects(spl):
    f = CASES[0].flux
    with pytest.raises(spl.SplidarError):
        spl.build_eq4(f, -1.0)
    with pytest.raises(spl.SplidarError):
        spl.build_eq4(f, float("nan"))
