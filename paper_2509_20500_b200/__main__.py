"""Command line front end of the B200 path (argument parsing and JSON output only; every step runs in
libsplidar.so). Exit codes: 0 ok, 2 invalid configuration, 3 power iteration
did not converge, 4 I/O error.

    python -m paper_2509_20500_b200 solve --t-r 100 --n-bins 256 --tau 40 --sigma 0.5 --signal 0.5 \\
        --background 0.1 --t-d 75 [--path dense|structured] [--dtype f64|f32] [--spectral] [--mixing] \\
        [--out result.json]
    python -m paper_2509_20500_b200 mc --t-r 100 --n-bins 1024 ... --t-d 75 --runs 100 --cycles 50000

Times in ns, S and B in photons per laser period; several --tau/--sigma/--signal values give
a multi-return flux (Eq. 1 summed over pulses)."""
from __future__ import annotations

import argparse
import json
import sys

EXIT_OK, EXIT_CONFIG, EXIT_NOCONV, EXIT_IO = 0, 2, 3, 4


class _Flux:
    def __init__(self, a):
        self.t_r = a.t_r
        self.n_bins = a.n_bins
        self.tau = tuple(a.tau)
        self.sigma = tuple(a.sigma)
        self.signal = tuple(a.signal)
        self.background = a.background


def _parser():
    p = argparse.ArgumentParser(prog="python -m paper_2509_20500_b200", description=__doc__.split("\n")[0])
    sub = p.add_subparsers(dest="cmd", required=True)
    for name in ("solve", "mc"):
        q = sub.add_parser(name)
        q.add_argument("--t-r", type=float, required=True, help="laser period t_r (ns)")
        q.add_argument("--n-bins", type=int, required=True, help="number of timestamp bins N")
        q.add_argument("--tau", type=float, nargs="+", required=True, help="pulse centre(s) (ns)")
        q.add_argument("--sigma", type=float, nargs="+", required=True, help="pulse width(s) (ns)")
        q.add_argument("--signal", type=float, nargs="+", required=True, help="signal photons / period per pulse")
        q.add_argument("--background", type=float, required=True, help="background photons / period")
        q.add_argument("--t-d", type=float, required=True, help="dead time (ns)")
        q.add_argument("--out", default=None, help="write the JSON result here (default: stdout)")
        if name == "solve":
            q.add_argument("--path", choices=["dense", "structured"], default="dense")
            q.add_argument("--dtype", choices=["f64", "f32"], default="f64")
            q.add_argument("--tol", type=float, default=1e-12)
            q.add_argument("--max-iter", type=int, default=10 ** 6)
            q.add_argument("--spectral", action="store_true", help="also lambda_2 (modulus, phase, gap)")
            q.add_argument("--mixing", action="store_true", help="also the mixing steps (eps 1e-3)")
        else:
            q.add_argument("--runs", type=int, default=100)
            q.add_argument("--cycles", type=int, default=50000)
            q.add_argument("--hist-bins", type=int, default=None, help="histogram bins (default N)")
            q.add_argument("--burn", type=int, default=100)
            q.add_argument("--seed", type=int, default=1)
    return p


def _emit(obj, path):
    text = json.dumps(obj)
    if path is None:
        print(text)
        return
    with open(path, "w") as f:
        f.write(text + "\n")


def main(argv=None) -> int:
    a = _parser().parse_args(argv)
    if not (len(a.tau) == len(a.sigma) == len(a.signal)):
        print("error: --tau, --sigma and --signal need the same number of values", file=sys.stderr)
        return EXIT_CONFIG
    import torch
    from . import splidar as spl
    f = _Flux(a)
    try:
        if a.cmd == "solve":
            status = EXIT_OK
            if a.path == "dense":
                dt = torch.float64 if a.dtype == "f64" else torch.float32
                P0 = spl.build_base(f, dt)
                pi, info = spl.stationary(P0, f.t_r, a.t_d, a.tol, a.max_iter, check=False)
                pi = pi.reshape(1, -1)
            else:
                shape, S, B = spl.flux_items(f)
                pi, infos = spl.stationary_structured(shape, S, B, [a.t_d], a.tol, a.max_iter, check=False)
                info = infos[0]
            if not info["converged"]:
                status = EXIT_NOCONV
            out = {"n_bins": f.n_bins, "shift_l": int(info["shift_l"]), "iters": int(info["iters"]),
                   "converged": bool(info["converged"]), "l1_change": float(info["l1_change"]), "path": a.path,
                   "pi": pi[0].cpu().tolist()}
            if a.spectral and status == EXIT_OK:
                if a.path == "dense":   # on the stored matrix (two-vector GEMV products)
                    l2 = spl.second_eigenvalue_dense(P0, f.t_r, a.t_d, pi[0].contiguous(), check=False)
                    l2 = dict(l2, lambda2_re=l2["lambda2"].real, lambda2_im=l2["lambda2"].imag)
                else:
                    shape, S, B = spl.flux_items(f)
                    l2 = spl.second_eigenvalue(shape, S, B, [a.t_d], pi.contiguous(), check=False)[0]
                out["lambda2"] = {"re": float(l2["lambda2_re"]), "im": float(l2["lambda2_im"]),
                                  "modulus": float(l2["modulus"]), "phase": float(l2["phase"]),
                                  "gap": float(l2["gap"]), "converged": bool(l2["converged"])}
            if a.mixing and status == EXIT_OK:
                n, _ = spl.mixing_steps(f, a.t_d, pi[0].contiguous(), check=False)
                out["mixing_steps"] = n
        else:
            shape, S, B = spl.flux_items(f)
            nh = a.hist_bins or f.n_bins
            h = spl.monte_carlo(shape, S, B, [a.t_d], a.seed, a.runs, nh, n_burn=a.burn, n_cycles=a.cycles)[0]
            counts = h.sum(dim=0).cpu()
            out = {"runs": a.runs, "cycles_per_run": a.cycles, "registrations": int(counts.sum()),
                   "histogram": counts.tolist(), "pdf": (counts.double() / counts.sum()).tolist()}
            status = EXIT_OK
    except spl.SplidarError as e:
        print(f"error: {e}", file=sys.stderr)
        return EXIT_NOCONV if e.status == spl.ENOCONV else EXIT_CONFIG
    try:
        _emit(out, a.out)
    except OSError as e:
        print(f"error: {e}", file=sys.stderr)
        return EXIT_IO
    return status


if __name__ == "__main__":
    sys.exit(main())
