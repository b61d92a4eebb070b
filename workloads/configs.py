"""BASELINE.json configs as concrete, seeded parameter sets (inputs only).

Units: times in ns (t_r, t_d, tau, sigma); S and B in mean photons per laser period
(S := alpha*E, B := t_r*lambda_b). A flux with K pulses generalises Eq. 1
 by summation; K = 1 is the paper's model.

Seeds (SURVEY §8(c) ambiguity 13-14):
  config 2: pulse centres  numpy.random.default_rng(0).uniform(10, 90, 6), in the order
            S in {0.1, 1, 5} (outer) x B in {0.01, 0.5} (inner).
  config 3: S = 10**U(-2, 1), B = 10**U(-3, log10 2), 64 pairs, default_rng(1), S drawn first.
  config 5: dead-time sweep numpy.linspace(10, 500, 16) (inclusive).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np


@dataclass(frozen=True)
class Flux:
    """theta without t_d: period t_r, N = n_b bins, K Gaussian pulses (tau, sigma, S), background B."""

    t_r: float
    n_bins: int
    tau: tuple
    sigma: tuple
    signal: tuple
    background: float

    @property
    def n_pulses(self) -> int:
        return len(self.tau)

    def scaled(self, eps: float) -> "Flux":
        """Same shape with every photon count multiplied by eps (vanishing-flux pin P4)."""
        return Flux(self.t_r, self.n_bins, self.tau, self.sigma,
                    tuple(eps * s for s in self.signal), eps * self.background)

    def with_bins(self, n: int) -> "Flux":
        return Flux(self.t_r, n, self.tau, self.sigma, self.signal, self.background)


@dataclass(frozen=True)
class Item:
    flux: Flux
    t_d: float


@dataclass
class Workload:
    name: str
    description: str
    items: list
    dtypes: tuple = ("f64",)
    sweep: list = field(default_factory=list)   # extra items sharing items[0].flux (config 5)

    @property
    def n_bins(self) -> int:
        return self.items[0].flux.n_bins


def _gauss(t_r, n, tau, sigma, signal, bg) -> Flux:
    return Flux(float(t_r), int(n), (float(tau),), (float(sigma),), (float(signal),), float(bg))


def config(k: int) -> Workload:
    """BASELINE.json configs[k-1] (k = 1..5)."""
    if k == 1:
        f = _gauss(100.0, 256, 40.0, 0.5, 0.5, 0.1)
        return Workload("c1", "N=256 t_r=100 fp64, pulse 40/0.5 S=0.5 B=0.1, t_d=75", [Item(f, 75.0)])
    if k == 2:
        centres = np.random.default_rng(0).uniform(10.0, 90.0, 6)
        items, c = [], 0
        for s in (0.1, 1.0, 5.0):
            for b in (0.01, 0.5):
                items.append(Item(_gauss(100.0, 1024, centres[c], 0.3, s, b), 50.0))
                c += 1
        return Workload("c2", "N=1024 t_r=100 fp64, 6 (S,B) pulses sigma 0.3, t_d=50", items)
    if k == 3:
        rng = np.random.default_rng(1)
        S = 10.0 ** rng.uniform(-2.0, 1.0, 64)
        B = 10.0 ** rng.uniform(-3.0, math.log10(2.0), 64)
        items = [Item(_gauss(100.0, 4096, 55.0, 0.2, s, b), 80.0) for s, b in zip(S, B)]
        return Workload("c3", "N=4096 t_r=100 fp64 batched sweep, 64 log-uniform (S,B), t_d=80", items)
    if k == 4:
        f = _gauss(100.0, 16384, 30.0, 0.1, 3.0, 1.0)
        return Workload("c4", "N=16384 t_r=100 fp64, pulse 30/0.1 S=3 B=1, t_d=120", [Item(f, 120.0)])
    if k == 5:
        f = Flux(200.0, 32768, (60.0, 140.0), (0.15, 0.15), (2.0, 0.5), 0.8)
        sweep = [Item(f, float(t)) for t in np.linspace(10.0, 500.0, 16)]
        return Workload("c5", "N=32768 t_r=200 fp64+fp32, two returns, B=0.8, t_d=430 + 16-value t_d sweep",
                        [Item(f, 430.0)], dtypes=("f64", "f32"), sweep=sweep)
    raise ValueError(f"no config {k}")


def all_configs() -> list:
    return [config(k) for k in range(1, 6)]


def random_flux(rng: np.random.Generator, n_bins: int, k_pulses: int = 1, t_r: float = 100.0,
                s_range=(0.01, 10.0), b_range=(0.001, 2.0), sigma_bins=(0.5, 20.0)) -> Flux:
    """Random flux shaped like the paper's workloads: narrow Gaussian returns on a flat floor
    (S, B log-uniform as config 3; sigma spanning 0.5-20 bins as configs 1-5 do)."""
    d = t_r / n_bins
    tau = tuple(float(x) for x in rng.uniform(0.1 * t_r, 0.9 * t_r, k_pulses))
    sig = tuple(float(x) for x in d * 10.0 ** rng.uniform(math.log10(sigma_bins[0]),
                                                           math.log10(sigma_bins[1]), k_pulses))
    S = tuple(float(x) for x in 10.0 ** rng.uniform(math.log10(s_range[0]), math.log10(s_range[1]), k_pulses))
    B = float(10.0 ** rng.uniform(math.log10(b_range[0]), math.log10(b_range[1])))
    return Flux(float(t_r), int(n_bins), tau, sig, S, B)


def parity_cases(seed: int = 7) -> list:
    """Small seeded (flux, t_d) cases for GPU-vs-oracle parity: several tiles, ragged tails,
    tiny N, exact-integer and fractional shifts, t_d beyond one period, K = 1 and 2 pulses."""
    rng = np.random.default_rng(seed)
    cases = []
    for n in (2, 3, 7, 64, 255, 1000, 1537, 2048):
        for kp in (1, 2):
            f = random_flux(rng, n, kp)
            td = float(rng.uniform(0.0, 3.0 * f.t_r))
            cases.append(Item(f, td))
    # exact integer shift u = x_d / Delta, whole periods, zero dead time
    f = random_flux(rng, 512, 1)
    cases += [Item(f, 0.0), Item(f, f.t_r), Item(f, 2.0 * f.t_r), Item(f, 75.0), Item(f, 37.5 + f.t_r)]
    return cases


def spectral_grid(n_bins: int = 256, n_side: int = 64, t_ds=(75.0, 95.0)) -> Workload:
    """Stand-in for the paper's (S, B) grids (Fig. 3c: S, B in [0, 10] at 2^8 bins; Fig. 4,
    P:187-191 and §4.2: t_d = 75 and 95): n_side x n_side (S, B) pairs on linspace(0.05, 10)
    (B > 0 keeps the chain irreducible, R16), one Gaussian return at 40 ns with
    sigma 0.5 ns (config 1's pulse), t_r = 100 ns, each pair at every t_d. Inputs only."""
    v = np.linspace(0.05, 10.0, n_side)
    items = []
    for td in t_ds:
        for s in v:
            for b in v:
                items.append(Item(_gauss(100.0, n_bins, 40.0, 0.5, float(s), float(b)), float(td)))
    return Workload("grid", f"(S,B) grid {n_side}x{n_side} on [0.05,10]^2 x t_d {list(t_ds)}, N={n_bins}, "
                            f"pulse 40/0.5, t_r=100", items)
