"""Seeded synthetic inputs shared by the oracle tests, the GPU parity tests and bench.py.

This package holds NO arithmetic of the method (no flux integrals, no matrix entries, no
shift rule): it only states the problem parameters theta = (t_r, t_d, sigma_t, tau, S, B, n_b)
(§2.3 "Distortion of Timestamp Distribution") for each BASELINE.json config and
for the small parity cases, drawing random ones from documented numpy PCG64 seeds.
"""
from .configs import Flux, Item, Workload, config, all_configs, parity_cases, random_flux, spectral_grid  # noqa: F401
