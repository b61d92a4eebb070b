"""Writes tests/golden/config1_oracle.json from the CPU oracle only (regression fixture, not a pin)."""
import json, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402
from workloads import config  # noqa: E402

it = config(1).items[0]
P = oracle.build_eq4(it.flux, it.t_d)
pi = oracle.stationary_dense(P)
rows = [0, 1, 100, 191, 192, 255]
out = {"source": "oracle.build_eq4 + oracle.stationary_dense, BASELINE config 1 (N=256, t_d=75)",
       "rows": {str(r): P[r].tolist() for r in rows}, "pi": pi.tolist()}
with open(os.path.join(ROOT, "tests", "golden", "config1_oracle.json"), "w") as f:
    json.dump(out, f)
print("wrote", len(pi))
