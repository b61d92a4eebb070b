"""The command line front end (python -m paper_2509_20500_b200): results vs the oracle and the exit
codes of SURVEY §8(b) / SPEC S:439 (0 ok, 2 invalid configuration, 3 no convergence, 4 I/O)."""
import json

import numpy as np
import pytest

import oracle
from workloads import config

C1 = ["--t-r", "100", "--n-bins", "256", "--tau", "40", "--sigma", "0.5", "--signal", "0.5",
      "--background", "0.1", "--t-d", "75"]


def _main(argv):
    from paper_2509_20500_b200.__main__ import main
    return main(argv)


def test_cli_rejects_mismatched_pulses():
    assert _main(["solve", "--t-r", "100", "--n-bins", "64", "--tau", "40", "50", "--sigma", "0.5",
                  "--signal", "1", "--background", "0.1", "--t-d", "10"]) == 2


@pytest.mark.gpu
@pytest.mark.parametrize("path", ["dense", "structured"])
def test_cli_solve_matches_oracle(tmp_path, path):
    out = tmp_path / "r.json"
    assert _main(["solve", *C1, "--path", path, "--spectral", "--mixing", "--out", str(out)]) == 0
    r = json.loads(out.read_text())
    it = config(1).items[0]
    P = oracle.build_eq4(it.flux, it.t_d)
    assert np.sum(np.abs(np.array(r["pi"]) - oracle.stationary_dense(P))) <= 1e-10
    assert r["shift_l"] == 192 and r["converged"]
    assert abs(r["lambda2"]["modulus"] - abs(oracle.second_eigenvalue(P))) <= 1e-8
    assert r["mixing_steps"] == oracle.mixing_steps(P, oracle.stationary_dense(P), 1e-3)[0]


@pytest.mark.gpu
def test_cli_exit_codes(tmp_path):
    assert _main(["solve", *C1, "--max-iter", "2", "--out", str(tmp_path / "a.json")]) == 3
    bad = [x if x != "0.1" else "0" for x in C1]                       # B = 0: invalid (R16)
    assert _main(["solve", *bad, "--out", str(tmp_path / "b.json")]) == 2
    assert _main(["solve", *C1, "--out", str(tmp_path / "missing_dir" / "c.json")]) == 4
    out = tmp_path / "mc.json"
    assert _main(["mc", *C1, "--runs", "8", "--cycles", "2000", "--hist-bins", "16", "--out", str(out)]) == 0
    r = json.loads(out.read_text())
    assert r["registrations"] == sum(r["histogram"]) > 0 and len(r["pdf"]) == 16
