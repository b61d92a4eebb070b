#!/usr/bin/env python
"""bench.py — throughput of the hot path of arXiv 2509.20500 on B200 (one JSON line on rank 0).

A step = one pass of the whole hot path over one batch of synthetic input: step 1-2 (flux vectors,
prefix sums, base matrix P~0 written to HBM) and step 3-4 (dead time folded into the gather,
power iteration to L1 change < 1e-12 on the device) for every item of the workload.

Default workload: BASELINE.json configs[4] ("c5"): N = 32768, t_r = 200 ns, two returns, fp64;
one P~0, the 16-value dead-time sweep plus the t_d = 430 ns solve on the same P~0, all 17 in one
multi-vector GEMV plan (each dead time its own gathered vector, Thm 2) = 17 stationary solves per step. --workload c1..c5 selects another config (c2, c3: batched items).

Metric (BASELINE.json): stationary solves/s (value, whole job), with transition-matrix entries/s,
and the fraction of the HBM roofline of the dominant kernel (the power-iteration GEMV) and of the
construction kernel. The 8.6 GB matrix is larger than the 126 MB L2, so no flush is needed between
steps (config.l2 says so). Device time by CUDA events on the launching stream; max over ranks.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload c5] [--dtype f64|f32]
                    [--mode factored|exp] [--impl ours|reference]
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METRIC = "stationary solves/s (with transition-matrix entries/s; % of HBM roofline)"
GEMV_KERNELS = {"tensor_i8": "k_power_step_i8 (tcgen05 kind::i8 exact split, TMEM accumulators)",
                "tensor_i8_encoded": "k_power_step_i8e (tcgen05 kind::i8 on encoded fp32 storage: TMA tiles are "
                                     "the MMA operand, TMEM accumulators)",
                "fp64": "k_power_step (FP64 tensor cores / DFMA)", "fused": "k_power_fused (cluster, small N)",
                "fp64_loop": "k_power_loop GEMV phase (FP64 tensor cores / DFMA; persistent GEMV + check kernel)"}
UNIT = "solves/s"


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=5)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--workload", default="c5", choices=["c1", "c2", "c3", "c4", "c5", "grid"])
    p.add_argument("--path", default="dense", choices=["dense", "structured", "spectral", "spectral_dense", "eq4",
                                                       "mc"],
                   help="dense: the north-star path (P~0 in HBM + GEMV power iteration); structured: "
                        "SURVEY f2 matrix-free solve; spectral: SURVEY f1 solve + lambda_2; eq4: SURVEY f4 "
                        "element-wise Eq. 4 construction (with Theorem 2's construction timed beside it); mc: "
                        "SURVEY f3 Monte Carlo of the detection process (paper protocol, P:202)")
    p.add_argument("--dtype", default="f64", choices=["f64", "f32"])
    p.add_argument("--mode", default="factored", choices=["factored", "exp"])
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--mc-split", type=int, default=None, help="--path mc: sub-chains per run (default: auto)")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-graph", action="store_true", help="dense path: never replay the step as a CUDA graph")
    p.add_argument("--shard", default="items", choices=["items", "rows"],
                   help="multi-GPU split (SURVEY 8(e)): items = independent items per rank, no collective (weak "
                        "scaling); rows = one matrix split by rows, one NCCL all-reduce of N x V doubles per "
                        "iteration (strong scaling; dense path, c4 / c5)")
    return p.parse_args()


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


# ------------------------------------------------------------------------------- workload
def workload_items(name, rank=0, world=1):
    """(Workload, groups): groups = [(flux, [dead times sharing that flux's P~0]), ...] for this rank.
    c5: every rank solves t_d = 430 and its 16-value shard of a 16 * world-point dead-time sweep over
    [10, 500] (world = 1: the config's own linspace(10, 500, 16)); other configs: every rank solves
    an independent replica of the config's items (weak scaling, no collective)."""
    from workloads import config, spectral_grid
    from paper_2509_20500_b200.shard import shard
    if name == "grid":
        w = spectral_grid()
        return w, [(it.flux, [it.t_d]) for it in shard(w.items, rank, world)]
    k = int(name[1])
    w = config(k)
    if k == 5:
        f = w.items[0].flux
        sweep = [float(t) for t in np.linspace(10.0, 500.0, 16 * world)]
        groups = [(f, shard(sweep, rank, world) + [w.items[0].t_d])]   # 17 dead times, one P~0, one plan
    else:
        groups = [(it.flux, [it.t_d]) for it in w.items]
    return w, groups


def load_traffic(workload, dtype):
    """dram bytes per launch of the dominant kernels from the committed ncu --set full capture."""
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            return json.load(f).get(f"{workload}_{dtype}")
    except Exception:
        return None


# ------------------------------------------------------------------------------- clocks
class ClockSampler:
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap,power.draw")

    def __init__(self, dev_index):
        self.proc = None
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                                          "-lms", "100", "-i", str(dev_index)], stdout=subprocess.PIPE,
                                         stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        out, _ = self.proc.communicate(timeout=10)
        sm, mx, reasons, pw = [], [], set(), []
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in out.strip().splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) < 7:
                continue
            try:
                sm.append(float(f[0]))
                mx.append(float(f[1]))
                pw.append(float(f[6]))
            except ValueError:
                continue
            for n, v in zip(names, f[2:6]):
                if v.lower() == "active":
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm), "power_w_max": max(pw) if pw else None}


# ------------------------------------------------------------------------------- our arm
class OurStep:
    def __init__(self, groups, dtype, mode):
        import torch
        import paper_2509_20500_b200 as spl
        self.spl, self.torch = spl, torch
        self.dt = torch.float64 if dtype == "f64" else torch.float32
        self.mode = mode
        self.N = groups[0][0].n_bins
        # one base matrix per distinct flux; each group = (flux, dead times sharing that P~0)
        fl, self.fluxes = [], []
        for f, tds in groups:
            if f not in fl:
                fl.append(f)
        self.fluxes = fl
        M = len(fl)
        self.P0 = spl.empty_matrix(self.N, self.dt, n_matrices=M)
        self.ws_build = spl.workspace(self.N, M, 1)
        self.plans = []
        # building plans: every launch runs steps 1-2 for its matrices and the power iteration, the
        # first product taken from the build's column sums (include/splidar.h: splidar_plan_create_build)
        if len(groups) == M and all(len(t) == 1 for _, t in groups):
            # one dead time per matrix (c1-c4): one plan over all M matrices
            tds = np.array([[t[0]] for _, t in groups])
            self.plans.append(spl.Plan(self.P0, fl[0].t_r, tds, tol=1e-12, build=fl, mode=mode))
        else:                    # c5: dead-time groups sharing a matrix, one multi-vector plan each
            for f, tds in groups:
                m = fl.index(f)
                self.plans.append(spl.Plan(self.P0[m], f.t_r, np.array([tds]), tol=1e-12, build=[f], mode=mode))
        self.n_solves = sum(len(t) for _, t in groups)
        self.entries = M * self.N * self.N

    def step(self):
        self.solve()             # the plans build their matrices

    def capture(self):
        """Small N (every plan fused = single launches): the whole step captured once as a CUDA graph and
        replayed, so a step is one cudaGraphLaunch instead of ~5 host API calls. Returns False otherwise."""
        torch = self.torch
        if not all(p.fused for p in self.plans):
            return False
        side = torch.cuda.Stream()
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):
            self.step()
        torch.cuda.current_stream().wait_stream(side)
        self.graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self.graph, capture_error_mode="thread_local"):
            self.step()
        self.graph_build = torch.cuda.CUDAGraph()      # the build alone, for the build / solve split
        with torch.cuda.graph(self.graph_build, capture_error_mode="thread_local"):
            self.build()
        return True

    def build(self):
        if len(self.fluxes) == 1:
            self.spl.build_base(self.fluxes[0], self.dt, self.mode, out=self.P0[0], ws=self.ws_build)
        else:
            self.spl.build_base_batched(self.fluxes, self.dt, self.mode, out=self.P0, ws=self.ws_build)

    def solve(self):
        for p in self.plans:
            p.launch()

    def infos(self):
        return [p.info() for p in self.plans]


def run_ours(args, rank, world, dev):
    import torch
    import paper_2509_20500_b200 as spl
    w, groups = workload_items(args.workload, rank, world)
    st = OurStep(groups, args.dtype, args.mode)
    stream = torch.cuda.current_stream()
    graphed = (not args.no_graph) and st.capture()
    for _ in range(args.warmup):
        if graphed:
            st.graph.replay()
        else:
            st.step()
    torch.cuda.synchronize()

    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True),
           torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    for p in st.plans:                   # the GEMV kernels' own device time over the timed region
        p.gemv_time(reset=True)
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    clocks = ClockSampler(dev)
    time.sleep(0.25)
    for e0, e1, e2 in ev:
        e0.record(stream)
        if graphed:                      # one replay = build + solve; the split is not observable
            st.graph.replay()
        else:                            # one launch per plan = build + solve (building plans)
            st.step()
        e2.record(stream)
    torch.cuda.synchronize()
    gtimes = [p.gemv_time() for p in st.plans]
    t_kernel = sum(t for t, _ in gtimes)
    n_kernel = sum(n for _, n in gtimes)
    # build share (build roofline): the same builds alone, timed after the steps
    if graphed:
        st.graph_build.replay()
    else:
        st.build()
    b0, b1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    b0.record(stream)
    for _ in range(len(ev)):
        if graphed:
            st.graph_build.replay()
        else:
            st.build()
    b1.record(stream)
    torch.cuda.synchronize()
    t_b = b0.elapsed_time(b1) / 1e3 / len(ev)
    if world > 1:
        torch.distributed.barrier()
    clk = clocks.stop()
    t_total = sum(a.elapsed_time(c) for a, _, c in ev) / 1e3
    t_build = min(t_b * len(ev), t_total)
    t_solve = t_total - t_build
    infos = st.infos()
    gemv_kinds = sorted({p.gemv() + ("_encoded" if p.gemv() == "tensor_i8" and p.storage() == "encoded" else "")
                         + ("_loop" if p.kind == "loop" else "") for p in st.plans})
    from paper_2509_20500_b200.shard import max_over_ranks
    t_total, t_build, t_solve, t_kernel = max_over_ranks([t_total, t_build, t_solve, t_kernel], device="cuda")

    b = 8 if args.dtype == "f64" else 4
    N = st.N
    # algorithmic GEMV bytes: every launch reads each still-active matrix once (N^2 b); launches =
    # iterations of the longest vector in each plan; matrices whose vectors all converged are skipped
    # (a building graph plan takes iteration 1 from the build's column sums: one GEMV launch fewer)
    launches_gemv, gemv_bytes = 0, 0
    for plan_info, p in zip(infos, st.plans):
        per_m = np.array([i["iters"] for i in plan_info]).reshape(p.M, p.V).max(axis=1)
        if not p.fused:
            per_m = np.maximum(per_m - 1, 0)
        launches_gemv += int(per_m.max())
        gemv_bytes += int(per_m.sum()) * N * N * b
    # every plan builds its matrices (fluxes stay in the plan's workspace: no upload): the step-1 vector
    # kernels (k_vec_small when N + 1 <= 8192, else k_vec_a..e) + k_build; encoded fp32 storage adds the
    # column-exponent pass before the build (k_enc_colexp + k_enc_flag). Then a fused plan is one launch;
    # a graph plan: column-sum reduce, init, ssum + check (iteration 1 from the column sums), GEMV + check
    # per further iteration, finish; int8 plans add the FP64 GEMV's early exit per iteration
    small = N + 1 <= 8192
    prelude = (1 if small else 5) + 1
    storages = [p.storage() for p in st.plans]

    def plan_launches(pi, p, storage):
        if p.fused:
            return prelude + 1
        it = int(np.array([i["iters"] for i in pi]).reshape(p.M, p.V).max())
        # the iterations after the first: GEMV + check each, or one persistent loop launch
        n = prelude + 1 + 1 + 2 + (1 if p.kind == "loop" else 2 * (it - 1)) + 1
        if p.gemv() == "tensor_i8":
            n += it - 1
        return n + (2 if storage == "encoded" else 0)
    per_step_launches = sum(plan_launches(pi, p, sg) for pi, p, sg in zip(infos, st.plans, storages))
    hbm, hbm_src = load_peaks()
    traffic = load_traffic(args.workload, args.dtype)
    K = args.steps
    gemv_gbs_phase = gemv_bytes * K / t_solve / 1e9
    # the kernel's own rate: algorithmic bytes / the GEMV launches' device time (graph plans); fused
    # plans have no separate GEMV kernel, so the solve phase stands in
    kernel_timed = n_kernel > 0 and n_kernel == launches_gemv * K
    gemv_gbs = gemv_bytes * K / t_kernel / 1e9 if kernel_timed else gemv_gbs_phase
    build_gbs = st.entries * b * K / t_build / 1e9
    units = st.n_solves * K * world
    value = units / t_total

    e2e = None
    if not args.no_e2e:
        e2e = run_e2e(args, w, groups, st, world)

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": K, "warmup": args.warmup,
        "ms_per_step": t_total / K * 1e3, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": args.dtype, "data": "synthetic (seeded BASELINE.json flux parameters; inputs are theta only)",
        "config": {"workload": f"{args.workload}: {w.description}", "n_bins": N,
                   "matrices_per_step": len(st.fluxes), "solves_per_step": st.n_solves, "entry_mode": args.mode,
                   "tol": 1e-12, "l2": "matrix (%.2f GB) > 126 MB L2: no flush needed" % (st.entries * b / 1e9)
                   if st.entries * b > 126e6 else "matrix fits in L2 (latency-bound config); not flushed",
                   "parallelism": (f"dp{world}: items sharded over {world} ranks, no collective on the data path"
                                   if world > 1 else "single GPU"),
                   "solver": "fused (one clustered launch per plan, N <= 2048)" if all(p.fused for p in st.plans)
                   else "loop (every iteration in one cooperative launch of the persistent GEMV + check kernel)"
                   if all(p.kind == "loop" for p in st.plans)
                   else "graph (GEMV + check in a conditional WHILE node)",
                   "gemv": gemv_kinds,
                   "step_as_cuda_graph": bool(graphed)},
        "entries_per_s": st.entries * K * world / t_build,
        "solves_per_s_solve_only": st.n_solves * K * world / t_solve,
        "paper_context": {"claim": "up to 1000x faster construction than Rapp's element-wise method",
                          "where": "abstract P:5, §3.5 P:199", "hardware": "not stated in the paper",
                          "same_gpu_ratio": "bench.py --path eq4 (Theorem 2 vs element-wise Eq. 4 on this B200)"},
        "ms_build_per_step": t_build / K * 1e3, "ms_solve_per_step": t_solve / K * 1e3,
        "iterations": [[i["iters"] for i in pi] for pi in infos],
        "roofline": {"bound": "hbm", "kernel": GEMV_KERNELS.get(gemv_kinds[0], gemv_kinds[0]) + " (power-iteration GEMV)"
                     if len(gemv_kinds) == 1 else "+".join(gemv_kinds), "achieved": gemv_gbs,
                     "peak": hbm, "unit": "GB/s", "frac": gemv_gbs / hbm,
                     "traffic": (traffic.get({"tensor_i8": "k_power_step_i8",
                                              "tensor_i8_encoded": "k_power_step_i8e"}.get(gemv_kinds[0], "k_power_step"))
                                 if traffic else None),
                     "algorithmic_bytes_per_launch": N * N * b,
                     "traffic_source": traffic.get("source") if traffic else None,
                     "peak_source": hbm_src,
                     "achieved_solve_phase": gemv_gbs_phase, "frac_solve_phase": gemv_gbs_phase / hbm,
                     "kernel_ms_per_launch": t_kernel / n_kernel * 1e3 if kernel_timed else None,
                     "kernel_launches": n_kernel,
                     "note": ("achieved = algorithmic bytes (N^2 b per launch per active matrix) / the GEMV "
                              "launches' own duration, measured on the device over the timed region (each launch, or each pass of the persistent loop kernel, "
                              "stamps %globaltimer at its first CTA's start and last CTA's end: "
                              "splidar_plan_gemv_time; CUDA events cannot bracket one kernel inside the graph's "
                              "WHILE loop); achieved_solve_phase divides by the whole solve phase (GEMV + check "
                              "kernels + graph loop)") if kernel_timed else
                             ("achieved = algorithmic bytes (N^2 b per launch per active matrix) / solve-phase "
                              "time (the fused solver has no separate GEMV kernel)")},
        "roofline_build": {"bound": "hbm", "kernel": "k_build", "achieved": build_gbs, "peak": hbm, "unit": "GB/s",
                           "frac": build_gbs / hbm, "traffic": traffic.get("k_build") if traffic else None,
                           "note": "N^2 b bytes written per matrix / build-phase time "
                                                            "(includes the flux-vector scan kernel)"},
        "clocks": clk, "e2e": e2e, "gpu_launches": per_step_launches * K,
        "impl": "ours", "lib": spl.lib_path(),
    }
    return line


def run_e2e(args, w, groups, st, world):
    """Same metric through the public Plan API a user re-solving with new parameters makes, with host
    buffers: theta from the host every step (Plan.set_fluxes), the building plan's launch (build +
    solve), pi copied to pinned host memory and Plan.info's one synchronisation."""
    import torch
    import paper_2509_20500_b200 as spl
    N = st.N
    n_solves = st.n_solves
    pi_host = torch.empty((n_solves, N), dtype=torch.float64, pin_memory=True)
    dt = st.dt
    h2d = 0
    for f, tds in groups:
        h2d += 8 * (3 * len(f.tau) + 3) + 8 * len(tds)
    one_per_matrix = len(groups) == len(st.fluxes) and all(len(t) == 1 for _, t in groups)

    def one():
        # theta host -> device every step (set_fluxes), build + solve (one launch per plan), pi to
        # pinned host memory, one synchronisation (Plan.info)
        row = 0
        for p in st.plans:
            fl = st.fluxes if one_per_matrix else [st.fluxes[st.plans.index(p)]]
            p.set_fluxes(fl)
            p.launch()
            n = p.M * p.V
            pi_host[row:row + n].copy_(p.pi.reshape(n, N), non_blocking=True)
            row += n
        for p in st.plans:
            p.info()

    for _ in range(max(1, args.warmup)):
        one()
    torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        one()
    torch.cuda.synchronize()
    dt_s = time.perf_counter() - t0
    from paper_2509_20500_b200.shard import max_over_ranks
    dt_s = max_over_ranks([dt_s], device="cuda")[0]
    return {"value": n_solves * args.steps * world / dt_s, "unit": UNIT, "h2d_bytes_per_step": h2d,
            "d2h_bytes_per_step": n_solves * N * 8,
            "note": "host wall clock; the public Plan API (set_fluxes: theta to the device, launch: build + solve, "
                    "pi copied to pinned host memory, info: one synchronisation) every step"}


# ------------------------------------------------------------------------------- row shards (8(e)(ii))
def run_rows(args, rank, world, dev):
    """One matrix split by rows over the ranks: rank g builds rows row_block(N, g, W)
    of P~0 and the power iteration all-reduces the N x V partial products once per iteration over NCCL
    (the gather offset is applied after the collective, in the replicated check). The workload is the
    config's own (c5: t_d = 430 + the 16-value sweep, 17 vectors; c4: one solve), so the total work is
    fixed: strong scaling. Device time by CUDA events around each step, max over ranks."""
    import torch
    import torch.distributed as dist
    import paper_2509_20500_b200 as spl
    from paper_2509_20500_b200.shard import max_over_ranks, row_block, sharded_solve
    w, groups = workload_items(args.workload, 0, 1)            # every rank: the whole item list
    if len(groups) != 1:
        raise SystemExit("--shard rows: one matrix per step (c4, c5)")
    f, tds = groups[0]
    N = f.n_bins
    dt = torch.float64 if args.dtype == "f64" else torch.float32
    r0, n = row_block(N, rank, world)
    ld = spl.leading_dim(N, dt)
    rows = torch.empty((n, ld), dtype=dt, device="cuda")[:, :N]
    ws_b = spl.workspace(N)
    plan = spl.ShardPlan(rows, r0, N, f.t_r, tds, tol=1e-12)
    reduce = (lambda t: dist.all_reduce(t, op=dist.ReduceOp.SUM)) if world > 1 else (lambda t: None)
    n_ar = [0]

    def counted(t):
        n_ar[0] += 1
        reduce(t)

    def step():
        spl.build_base_rows(f, r0, n, dt, args.mode, out=rows, ws=ws_b)
        return sharded_solve(plan, counted)

    for _ in range(args.warmup):
        infos = step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clocks = ClockSampler(dev)
    time.sleep(0.25)
    stream = torch.cuda.current_stream()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    n_ar[0] = 0
    for e0, e1 in ev:
        e0.record(stream)
        infos = step()
        e1.record(stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clk = clocks.stop()
    K = args.steps
    ar_per_step = n_ar[0] // K
    t_total = max_over_ranks([sum(a.elapsed_time(b) for a, b in ev) / 1e3], device="cuda")[0]
    iters = [i["iters"] for i in infos]
    b = 8 if args.dtype == "f64" else 4
    passes = max(iters)
    hbm, hbm_src = load_peaks()
    # every rank reads its n x N block once per pass: the job reads N^2 b per pass
    gemv_gbs = passes * N * N * b * K / t_total / 1e9
    pi_host = torch.empty((len(tds), N), dtype=torch.float64, pin_memory=True)
    t0 = time.perf_counter()                           # e2e: theta from the host, pi to pinned host memory
    for _ in range(K):
        step()
        pi_host.copy_(plan.pi, non_blocking=True)
        torch.cuda.current_stream().synchronize()
    t_e2e = max_over_ranks([time.perf_counter() - t0], device="cuda")[0]
    value = len(tds) * K / t_total
    return {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": K, "warmup": args.warmup,
        "ms_per_step": t_total / K * 1e3, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": args.dtype, "data": "synthetic (seeded BASELINE.json flux parameters; inputs are theta only)",
        "config": {"workload": f"{args.workload}: {w.description}", "n_bins": N, "solves_per_step": len(tds),
                   "parallelism": f"rows{world}: P~0 split by rows over {world} ranks, one NCCL all-reduce of "
                                  f"N x {len(tds)} fp64 per iteration" if world > 1 else "single GPU (row shard of 1)",
                   "rows_per_rank": n, "allreduces_per_step": ar_per_step,
                   "l2": "matrix > 126 MB L2: no flush needed" if N * N * b > 126e6 else "fits in L2"},
        "iterations": iters,
        "roofline": {"bound": "hbm", "kernel": "k_power_step (row shard) + NCCL all-reduce", "achieved": gemv_gbs,
                     "peak": hbm * world, "unit": "GB/s", "frac": gemv_gbs / (hbm * world),
                     "traffic": None, "peak_source": hbm_src + f" x {world} GPUs",
                     "note": "job-wide algorithmic bytes (N^2 b per pass) / step time (build, GEMV, all-reduce, "
                             "check, host loop)"},
        "clocks": clk,
        "e2e": {"value": len(tds) * K / t_e2e, "unit": UNIT, "h2d_bytes_per_step": 8 * (3 * len(f.tau) + 3 + len(tds)),
                "d2h_bytes_per_step": len(tds) * N * 8},
        "gpu_launches": K * (2 + 5 + 1 + 3 * passes + 1), "impl": "ours", "lib": spl.lib_path(),
    }


# ------------------------------------------------------------------------------- stored-matrix lambda_2
def run_spectral_dense(args, rank, world, dev):
    """f1 on a stored matrix: per step, build the workload's first P~0, its stationary pi (dense GEMV
    plan) and lambda_2 by the two-vector GEMV subspace iteration (splidar_second_eigenvalue_dense).
    Roofline: the two-vector GEMV, N^2 b bytes per product (timed by CUDA events around the lambda_2
    call: products x bytes / that time, a lower bound on the kernel's own rate)."""
    import torch
    import paper_2509_20500_b200 as spl
    w, groups = workload_items(args.workload, rank, world)
    f, td = w.items[0].flux, w.items[0].t_d              # the workload's own item (c5: t_d = 430)
    N = f.n_bins
    dt = torch.float64 if args.dtype == "f64" else torch.float32
    b = 8 if args.dtype == "f64" else 4
    P0 = spl.empty_matrix(N, dt)
    ws_b = spl.workspace(N, 1, 1)
    from paper_2509_20500_b200 import splidar as _binding
    nb = _binding._lib().splidar_spectral_dense_workspace_bytes(N)
    t_ws = torch.empty(nb + 256, dtype=torch.uint8, device="cuda")
    ws_l2 = t_ws[(-t_ws.data_ptr()) % 256:][:nb]
    plan = spl.Plan(P0, f.t_r, [[td]], tol=1e-12)
    stream = torch.cuda.current_stream()
    res = {}

    def step():
        spl.build_base(f, dt, out=P0, ws=ws_b)
        plan.launch()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        res["l2"] = spl.second_eigenvalue_dense(P0, f.t_r, td, plan.pi[0, 0], ws=ws_l2)
        e1.record(stream)
        res["ev"] = (e0, e1)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    pinfo = plan.info()                                  # raises unless pi converged
    if not res["l2"]["converged"]:
        raise SystemExit("spectral_dense: lambda_2 did not converge")
    if world > 1:
        torch.distributed.barrier()
    clocks = ClockSampler(dev)
    time.sleep(0.25)
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    l2_ms = []
    t_total = 0.0
    for _ in range(args.steps):
        t0.record(stream)
        step()
        t1.record(stream)
        torch.cuda.synchronize()
        t_total += t0.elapsed_time(t1) / 1e3
        l2_ms.append(res["ev"][0].elapsed_time(res["ev"][1]))
    clk = clocks.stop()
    from paper_2509_20500_b200.shard import max_over_ranks
    t_total = max_over_ranks([t_total], device="cuda")[0]
    info = res["l2"]
    K = args.steps
    l2_s = statistics.mean(l2_ms) / 1e3
    achieved = info["iters"] * N * N * b / l2_s / 1e9
    hbm, hbm_src = load_peaks()
    return {
        "metric": "spectral analyses/s on a stored matrix (pi + lambda_2; SURVEY f1 via the multi-vector GEMV)",
        "value": world * K / t_total, "unit": "analyses/s", "n_gpus": world, "steps": K, "warmup": args.warmup,
        "ms_per_step": t_total / K * 1e3, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": args.dtype, "data": "synthetic (seeded BASELINE.json flux parameters)",
        "config": {"workload": f"{args.workload}: {w.description}", "n_bins": N, "t_d": td,
                   "step": "build P~0 + dense pi (GEMV plan) + lambda_2 (two-vector GEMV subspace iteration)",
                   "l2": "matrix > L2 for N >= 4096" if N * N * b > 126e6 else "L2-resident"},
        "lambda2": {"modulus": info["modulus"], "phase": info["phase"], "iters": info["iters"],
                    "converged": info["converged"]},
        "roofline": {"bound": "hbm", "kernel": "k_power_step<T, 2>", "achieved": achieved, "peak": hbm,
                     "unit": "GB/s", "frac": achieved / hbm, "traffic": None, "peak_source": hbm_src,
                     "algorithmic_bytes_per_launch": N * N * b, "lambda2_ms_per_step": statistics.mean(l2_ms)},
        "clocks": clk, "e2e": None,
        # build: (flux upload unless one small profile) + vectors + k_build; pi plan: one fused launch, or
        # init + (GEMV + check) per iteration + finish; lambda_2: init + 3 per product
        "gpu_launches": K * ((0 if N + 1 <= 8192 else 1) + (1 if N + 1 <= 8192 else 5) + 1
                             + (1 if plan.fused else 2 + 2 * int(pinfo[0]["iters"]))
                             + 1 + 3 * int(info["iters"])),
        "impl": "ours", "lib": spl.lib_path(),
    }


# ------------------------------------------------------------------------------- structured paths
FP64_PEAK_TFLOPS = 148 * 64 * 2 * 1.965e9 / 1e12   # 148 SMs x 64 DFMA/clk x 2 flop x 1.965 GHz
FLOPS_PER_ELEM = {"solve": 9, "lambda2": 48}      # algorithmic fp64 flops per bin per product


def _shape_groups(groups):
    """Items -> plans: one plan per pulse shape (t_r, N, tau, sigma, relative weights); items carry
    (S = total signal, B, t_d)."""
    from workloads import Flux
    plans = {}
    for f, tds in groups:
        tot = float(sum(f.signal))
        rel = tuple(x / tot for x in f.signal) if tot > 0 else tuple(f.signal)
        key = (f.t_r, f.n_bins, tuple(f.tau), tuple(f.sigma), rel)
        shape = Flux(f.t_r, f.n_bins, f.tau, f.sigma, rel, 1.0)
        e = plans.setdefault(key, [shape, [], [], []])
        for td in tds:
            e[1].append(tot if tot > 0 else 1.0)
            e[2].append(f.background)
            e[3].append(td)
    return list(plans.values())


def run_struct(args, rank, world, dev):
    import torch
    import paper_2509_20500_b200 as spl
    w, groups = workload_items(args.workload, rank, world)
    kind = "solve" if args.path == "structured" else "lambda2"
    sg = _shape_groups(groups)
    N = groups[0][0].n_bins
    solve_plans, l2_plans = [], []
    for shape, S, B, T in sg:
        sp = spl.StructPlan("solve", shape, S, B, T)
        solve_plans.append(sp)
        if kind == "lambda2":
            l2_plans.append(spl.StructPlan("lambda2", shape, S, B, T, pi=sp.pi))
    n_items = sum(len(g[1]) for g in sg)
    stream = torch.cuda.current_stream()

    def step():
        for p in solve_plans:
            p.launch()
        for p in l2_plans:
            p.launch()

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    clocks = ClockSampler(dev)
    time.sleep(0.25)
    t_total, k_ms, products = 0.0, [], 0
    main_plans = l2_plans if kind == "lambda2" else solve_plans
    for _ in range(args.steps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        step()
        e1.record(stream)
        torch.cuda.synchronize()
        t_total += e0.elapsed_time(e1) / 1e3
        ms = 0.0
        products = 0
        for p in main_plans:
            infos, kms = p.info()
            ms += kms
            products += int(infos["iters"].sum())
        k_ms.append(ms)
    if world > 1:
        torch.distributed.barrier()
    clk = clocks.stop()
    from paper_2509_20500_b200.shard import max_over_ranks
    t_total = max_over_ranks([t_total], device="cuda")[0]
    K = args.steps
    kernel_s = statistics.mean(k_ms) / 1e3
    flops = FLOPS_PER_ELEM[kind] * N * products
    achieved = flops / kernel_s / 1e12
    iters = [[int(x) for x in p.info()[0]["iters"]] for p in main_plans]
    conv = bool(all(int(x) for p in main_plans for x in p.info(check=False)[0]["converged"]))
    unit = "solves/s" if kind == "solve" else "spectral analyses/s"
    metric = ("stationary solves/s, matrix-free structured operator (SURVEY f2)" if kind == "solve" else
              "spectral analyses/s (pi + lambda_2, modulus and phase; SURVEY f1)")
    e2e = None if args.no_e2e else run_struct_e2e(args, sg, kind, world)
    return {
        "metric": metric, "value": n_items * K * world / t_total, "unit": unit, "n_gpus": world, "steps": K,
        "warmup": args.warmup, "ms_per_step": t_total / K * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded BASELINE.json flux parameters / (S, B) grid)",
        "config": {"workload": f"{args.workload}: {w.description}", "n_bins": N, "items_per_step": n_items,
                   "path": args.path, "tol": 1e-12 if kind == "solve" else 1e-13,
                   "l2": "no matrix is stored; per-item state lives in shared memory / registers",
                   "parallelism": "single GPU" if world == 1 else f"dp{world}: items sharded, no collective"},
        "converged": conv, "products_per_step": products,
        "iterations_max": max(max(x) for x in iters), "iterations_sum": sum(sum(x) for x in iters),
        "roofline": {"bound": "alu", "kernel": "k_struct_lambda2" if kind == "lambda2" else
                     ("k_struct_solve_c1" if N > 4096 else "k_struct_solve"),
                     "achieved": achieved, "peak": FP64_PEAK_TFLOPS, "unit": "TFLOP/s",
                     "frac": achieved / FP64_PEAK_TFLOPS, "traffic": None,
                     "algorithmic_flops_per_bin_product": FLOPS_PER_ELEM[kind],
                     "kernel_ms_per_step": statistics.mean(k_ms),
                     "peak_source": "derived: 148 SMs x 64 FP64 FMA/clk x 2 x 1.965 GHz (probe: 35.8 TFLOP/s DFMA)",
                     "note": "FP64 issue is not the limiter: per-product barriers, scan latency and instruction "
                             "issue are (DESIGN.md)"},
        "clocks": clk, "e2e": e2e,
        # per plan launch: the step-1 vector kernels (k_vec_small: 1 when N + 1 <= 8192, else k_vec_a..e: 5)
        # and the team kernel
        "gpu_launches": (len(main_plans) + (len(solve_plans) if kind == "lambda2" else 0))
                        * ((1 if N + 1 <= 8192 else 5) + 1) * K,
        "impl": "ours", "lib": spl.lib_path(),
    }


def run_struct_e2e(args, sg, kind, world):
    """Through the public one-shot calls with host theta and the results copied to pinned host memory."""
    import torch
    import paper_2509_20500_b200 as spl
    n = sum(len(g[1]) for g in sg)
    N = sg[0][0].n_bins
    pi_host = torch.empty((n, N), dtype=torch.float64, pin_memory=True)

    def one():
        row = 0
        for shape, S, B, T in sg:
            pi, _ = spl.stationary_structured(shape, S, B, T)
            if kind == "lambda2":
                spl.second_eigenvalue(shape, S, B, T, pi)
            pi_host[row:row + len(S)].copy_(pi, non_blocking=True)
            row += len(S)
        torch.cuda.current_stream().synchronize()

    for _ in range(max(1, args.warmup)):
        one()
    if world > 1:
        torch.distributed.barrier()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        one()
    dt_s = time.perf_counter() - t0
    from paper_2509_20500_b200.shard import max_over_ranks
    dt_s = max_over_ranks([dt_s], device="cuda")[0]
    h2d = sum(8 * (3 * len(shape.tau) + 1) + 24 * len(S) for shape, S, B, T in sg)
    return {"value": n * args.steps * world / dt_s, "unit": "solves/s" if kind == "solve" else "spectral analyses/s",
            "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": n * N * 8 + (n * 48 if kind == "lambda2" else 0),
            "note": "host wall clock; validation, grouping and upload of theta, kernels, pi to pinned host memory"}


def run_eq4(args, rank, world, dev):
    """P~ element by element from Eq. 4 for every item of the workload (its own dead time), and
    in the same run Theorem 2's construction of the same matrices (base matrix + materialised row
    permutation) for the same-hardware speed-up (the paper's Fig. 3a comparison)."""
    import torch
    import paper_2509_20500_b200 as spl
    w, groups = workload_items(args.workload, rank, world)
    items = [(f, td) for f, tds in groups for td in tds][:4 if args.workload == "c5" else None]
    N = items[0][0].n_bins
    dt = torch.float64 if args.dtype == "f64" else torch.float32
    b = 8 if args.dtype == "f64" else 4
    P = spl.empty_matrix(N, dt)
    P0 = spl.empty_matrix(N, dt)
    ws = spl.workspace(N)
    stream = torch.cuda.current_stream()

    def eq4_step():
        for f, td in items:
            spl.build_eq4(f, td, dt, out=P)

    def thm2_step():
        for f, td in items:
            spl.build_base(f, dt, args.mode, out=P0, ws=ws)
            spl.apply_deadtime(P0, f.t_r, td, out=P)

    def timed(fn):
        for _ in range(args.warmup):
            fn()
        torch.cuda.synchronize()
        evs = []
        for _ in range(args.steps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            fn()
            e1.record(stream)
            evs.append((e0, e1))
        torch.cuda.synchronize()
        return sum(a.elapsed_time(c) for a, c in evs) / 1e3

    if world > 1:
        torch.distributed.barrier()
    clocks = ClockSampler(dev)
    time.sleep(0.25)
    t_eq4 = timed(eq4_step)
    clk = clocks.stop()
    t_thm2 = timed(thm2_step)
    from paper_2509_20500_b200.shard import max_over_ranks
    t_eq4, t_thm2 = max_over_ranks([t_eq4, t_thm2], device="cuda")
    K = args.steps
    entries = len(items) * N * N
    traffic = load_traffic(args.workload + "_eq4", args.dtype) or {}
    flops_per_entry = traffic.get("fp64_flops_per_entry")
    achieved = flops_per_entry * entries * K / t_eq4 / 1e12 if flops_per_entry else None
    return {
        "metric": "transition-matrix entries/s, element-wise Eq. 4 construction (SURVEY f4)",
        "value": entries * K * world / t_eq4, "unit": "entries/s", "n_gpus": world, "steps": K,
        "warmup": args.warmup, "ms_per_step": t_eq4 / K * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": args.dtype, "data": "synthetic (seeded BASELINE.json flux parameters)",
        "config": {"workload": f"{args.workload}: {w.description}", "n_bins": N, "matrices_per_step": len(items),
                   "path": "eq4", "l2": "matrix > L2 for N >= 4096 (not flushed otherwise)",
                   "parallelism": "single GPU" if world == 1 else f"dp{world}"},
        "theorem2_same_gpu": {"entries_per_s": entries * K * world / t_thm2, "ms_per_step": t_thm2 / K * 1e3,
                              "what": "splidar_build_base + splidar_apply_deadtime (materialised J_l) per item",
                              "speedup_vs_eq4": t_eq4 / t_thm2},
        "paper_speedup_context": "up to 1000x vs Rapp's element-wise construction (P:5, P:199; hardware not stated)",
        "roofline": {"bound": "alu", "kernel": "k_build_eq4", "achieved": achieved, "peak": FP64_PEAK_TFLOPS,
                     "unit": "TFLOP/s", "frac": achieved / FP64_PEAK_TFLOPS if achieved else None,
                     "traffic": traffic.get("dram_bytes"),
                     "algorithmic_flops_per_entry": flops_per_entry,
                     "fp64_pipe_pct_ncu": traffic.get("fp64_pipe_pct"),
                     "flops_source": traffic.get("source"),
                     "peak_source": "derived: 148 SMs x 64 FP64 FMA/clk x 2 x 1.965 GHz (probe: 35.8 TFLOP/s DFMA)"},
        "clocks": clk, "e2e": None, "gpu_launches": len(items) * K, "impl": "ours", "lib": spl.lib_path(),
    }


def run_mc(args, rank, world, dev):
    """the paper's Monte Carlo protocol on the GPU. c1..c5: every item, 100 runs of 50,000
    laser cycles each, histograms at 2^10 bins; grid: a 16 x 16 (S, B) x {75, 95} grid at 2^8
    bins, 25 runs of 50,000 cycles per item. Metric: registrations/s."""
    import torch
    import paper_2509_20500_b200 as spl
    from workloads import spectral_grid
    if args.workload == "grid":
        w = spectral_grid(256, 16)
        groups = [(it.flux, [it.t_d]) for it in w.items]
        n_runs, n_hist = 25, 256
    else:
        w, groups = workload_items(args.workload, rank, world)
        n_runs, n_hist = 100, 1024
    sg = _shape_groups(groups)
    n_cycles, n_burn = 50000, 100
    n_items = sum(len(g[1]) for g in sg)
    # sub-chains per run for occupancy (~200k threads), each >= 3000 cycles; 1 = one chain per histogram
    n_split = max([d for d in range(1, 51) if n_cycles % d == 0 and n_cycles // d >= 3000
                   and d * n_items * n_runs <= max(200000, n_items * n_runs)] or [1])
    if args.mc_split is not None:
        n_split = args.mc_split
    stream = torch.cuda.current_stream()
    seed = [1000 + 7919 * rank]

    def step():
        regs = 0
        for shape, S, B, T in sg:
            h = spl.monte_carlo(shape, S, B, T, seed[0], n_runs, n_hist, n_burn=n_burn, n_cycles=n_cycles,
                                n_split=n_split)
            regs += h.sum()
        seed[0] += 1
        return regs

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    clocks = ClockSampler(dev)
    time.sleep(0.25)
    regs_t = []
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        regs_t.append(step())
    e1.record(stream)
    torch.cuda.synchronize()
    clk = clocks.stop()
    t_total = e0.elapsed_time(e1) / 1e3
    from paper_2509_20500_b200.shard import max_over_ranks
    t_total = max_over_ranks([t_total], device="cuda")[0]
    regs = int(sum(int(r) for r in regs_t))
    K = args.steps
    traffic = load_traffic(args.workload + "_mc", "f64") or {}
    fpr = traffic.get("fp64_flops_per_registration")
    achieved = fpr * regs / t_total / 1e12 if fpr else None
    return {
        "metric": "simulated registrations/s, Monte Carlo of the detection process (SURVEY f3)",
        "value": regs * world / t_total, "unit": "registrations/s", "n_gpus": world, "steps": K,
        "warmup": args.warmup, "ms_per_step": t_total / K * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded counter-based generator)",
        "config": {"workload": f"{args.workload}: {w.description}", "items": n_items, "runs_per_item": n_runs,
                   "laser_cycles_per_run": n_cycles, "n_hist": n_hist, "burn_in": n_burn, "path": "mc",
                   "n_split": n_split, "split_note": "each run = n_split independent sub-chains of n_cycles / n_split "
                                                     "cycles after their own burn-in, into one histogram",
                   "protocol": "P:202 (100 x 50,000 cycles, 2^10 bins)" if args.workload != "grid"
                   else "P:205 (25 x 50,000 cycles per (S, B), 2^8 bins)",
                   "parallelism": "single GPU" if world == 1 else f"dp{world}: chains seeded per rank"},
        "laser_cycles_per_s": n_items * n_runs * n_cycles * K * world / t_total,
        "registrations_per_step": regs / K,
        "roofline": {"bound": "alu", "kernel": "k_mc", "achieved": achieved, "peak": FP64_PEAK_TFLOPS,
                     "unit": "TFLOP/s", "frac": achieved / FP64_PEAK_TFLOPS if achieved else None,
                     "traffic": traffic.get("dram_bytes"), "algorithmic_flops_per_registration": fpr,
                     "fp64_pipe_pct_ncu": traffic.get("fp64_pipe_pct"),
                     "flops_source": traffic.get("source"),
                     "note": "time includes the host call (validation, uploads, histogram zeroing)",
                     "peak_source": "derived: 148 SMs x 64 FP64 FMA/clk x 2 x 1.965 GHz (probe: 35.8 TFLOP/s DFMA)"},
        "clocks": clk, "e2e": None, "gpu_launches": len(sg) * K, "impl": "ours", "lib": spl.lib_path(),
    }


def run_oracle_mc(args):
    """The oracle's single-chain Monte Carlo for about 10 s on one core of the host."""
    import oracle
    from workloads import spectral_grid
    if args.workload == "grid":
        f, td = spectral_grid(256, 16).items[0].flux, 75.0
    else:
        w, groups = workload_items(args.workload)
        f, td = groups[0][0], groups[0][1][0]
    n = 20000
    t0 = time.perf_counter()
    done = 0
    while time.perf_counter() - t0 < 10.0:
        oracle.monte_carlo(f, td, 1 + done, 0, n, 1, 256)
        done += n
    dt = time.perf_counter() - t0
    return {"value": done / dt, "unit": "registrations/s", "cores": 1, "kind": "oracle",
            "sample": f"{args.workload}: chains of {n} registrations (oracle_mc, bisection inversion), ~10 s"}


def run_oracle_spectral(args):
    """Oracle for the spectral path: Eq. 4 matrix, dense pi and numpy eigvals, on a bounded sample."""
    import oracle
    w, groups = workload_items(args.workload)
    N = groups[0][0].n_bins
    if N > 2048:
        return None
    t0 = time.perf_counter()
    n = 0
    for f, tds in groups:
        for td in tds:
            P = oracle.build_eq4(f, td)
            oracle.stationary_dense(P)
            oracle.second_eigenvalue(P)
            n += 1
            if time.perf_counter() - t0 > 10.0:
                break
        if time.perf_counter() - t0 > 10.0:
            break
    dt = time.perf_counter() - t0
    return {"value": n / dt, "unit": "spectral analyses/s", "cores": os.cpu_count(), "kind": "oracle",
            "sample": f"{args.workload}: {n} items (Eq. 4 matrix with OpenMP rows, dense Gaussian-elimination pi, "
                      f"numpy.linalg.eigvals), about 10 s"}


# ------------------------------------------------------------------------------- oracle arm
def host_info() -> dict:
    """CPU model, logical cores and RAM of the host the oracle runs on."""
    model, ram = None, None
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
        for line in open("/proc/meminfo"):
            if line.startswith("MemTotal"):
                ram = f"{int(line.split()[1]) / 1048576:.0f} GiB"
                break
    except OSError:
        pass
    return {"cpu_model": model, "logical_cores": os.cpu_count(), "ram": ram}


def run_oracle_sample(args, iters_per_item=None):
    """The CPU oracle as it stands on a bounded sample of the same workload: R rows of the Eq. 4
    matrix (OpenMP over rows) and the oracle's long-double product over them; scaled to whole
    solves. The oracle has no permutation trick, so it builds one Eq. 4 matrix per dead time."""
    import oracle
    w, groups = workload_items(args.workload)
    N = groups[0][0].n_bins
    R = min(N, 1024 if N >= 16384 else (2048 if N >= 4096 else N))
    rng = np.random.default_rng(0)
    t_build_row, t_mv_row = [], []
    for f, tds in groups[:4]:
        r0 = int(rng.integers(0, N - R + 1))
        t0 = time.perf_counter()
        rows = oracle.rows_eq4(f, tds[0], r0, r0 + R)
        t_build_row.append((time.perf_counter() - t0) / R)
        x = np.full(R, 1.0 / N)
        t0 = time.perf_counter()
        oracle.left_matvec(rows, x)
        t_mv_row.append((time.perf_counter() - t0) / R)
    tb, tm = statistics.median(t_build_row), statistics.median(t_mv_row)
    # the build's rows again on one thread (the OpenMP figure above uses every core)
    f0, tds0 = groups[0]
    oracle.set_threads(1)
    t0 = time.perf_counter()
    oracle.rows_eq4(f0, tds0[0], 0, min(R, 256))
    tb1 = (time.perf_counter() - t0) / min(R, 256)
    oracle.set_threads(os.cpu_count() or 1)
    total = 0.0
    n = 0
    for gi, (f, tds) in enumerate(groups):
        for vi, _ in enumerate(tds):
            its = iters_per_item[gi][vi] if iters_per_item else 25
            total += N * tb + its * N * tm
            n += 1
    cores = os.cpu_count()
    return {"value": n / total, "unit": UNIT, "cores": cores, "kind": "oracle",
            "sample": f"{args.workload}: {R} of {N} rows of Eq. 4 (OpenMP, {cores} threads) and one long-double "
                      f"product over them (1 thread), for up to 4 items; scaled to {n} full solves "
                      f"(N rows each, one Eq. 4 matrix per dead time, GPU iteration counts)",
            "s_per_row_build": tb, "s_per_row_product": tm,
            "build_entries_per_s_all_cores": N / tb, "build_entries_per_s_one_core": N / tb1,
            "solve_products_entries_per_s_one_core": N / tm, "host": host_info()}


def _free_port() -> int:
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def main():
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # not started by torchrun: launch one rank per GPU ourselves (rank 0 prints the line)
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), os.path.abspath(__file__),
               *sys.argv[1:]]
        return subprocess.call(cmd)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}", file=sys.stderr)
        return 2

    if args.impl == "reference":
        if rank != 0:
            return 0
        # W untimed warm-up steps, then K timed ones; a step is one bounded sample of the workload
        # (~2 s at c5: 1024 of N rows of up to 4 of the step's Eq. 4 matrices and their products).
        # ms_per_step is a sample's wall time; the value scales the sample to whole solves (median)
        for _ in range(max(0, args.warmup)):
            run_oracle_sample(args)
        samples, walls = [], []
        for _ in range(max(1, args.steps)):
            t0 = time.perf_counter()
            samples.append(run_oracle_sample(args))
            walls.append(time.perf_counter() - t0)
        v = statistics.median(s["value"] for s in samples)
        w, groups_ref = workload_items(args.workload)
        n_step = sum(len(t) for _, t in groups_ref)
        cb = dict(samples[0])
        cb["value"] = v
        line = {"metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus, "steps": len(samples),
                "warmup": max(0, args.warmup), "ms_per_step": 1e3 * statistics.median(walls),
                "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
                "dtype": args.dtype, "data": "synthetic", "impl": "reference",
                "config": {"workload": f"{args.workload}: {w.description}", "n_bins": w.n_bins},
                "step_note": ("a step is one bounded sample of the workload (cpu_baseline.sample); value = the "
                              f"sample scaled to whole solves (one full step of {n_step} solves would take "
                              f"{n_step / v:.0f} s on these cores)"),
                "cpu_baseline": cb, "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0,
                                             "d2h_bytes_per_step": 0}}
        print(json.dumps(line))
        return 0

    import torch
    if world > 1:
        torch.cuda.set_device(local)
        torch.distributed.init_process_group("nccl")
    else:
        torch.cuda.set_device(0)
    dev = torch.cuda.current_device()
    if args.path == "dense" and args.shard == "rows":
        line = run_rows(args, rank, world, dev)
    elif args.path == "dense":
        line = run_ours(args, rank, world, dev)
        if rank == 0 and world == 1 and not args.no_cpu_baseline:
            its = line["iterations"]
            if len(its) == 1 and len(its[0]) > 1 and args.workload != "c5":
                its = [[x] for x in its[0]]          # one plan over M matrices -> one list per item
            line["cpu_baseline"] = run_oracle_sample(args, its)
    elif args.path == "mc":
        line = run_mc(args, rank, world, dev)
        if rank == 0 and world == 1 and not args.no_cpu_baseline:
            line["cpu_baseline"] = run_oracle_mc(args)
    elif args.path == "spectral_dense":
        line = run_spectral_dense(args, rank, world, dev)
    elif args.path == "eq4":
        line = run_eq4(args, rank, world, dev)
        if rank == 0 and world == 1 and not args.no_cpu_baseline:
            cb = run_oracle_sample(args)
            w_, g_ = workload_items(args.workload)
            Nn = g_[0][0].n_bins
            cb = {"value": Nn / cb["s_per_row_build"], "unit": "entries/s", "cores": cb["cores"], "kind": "oracle",
                  "sample": cb["sample"].split(" and one")[0] + " (build only)"}
            line["cpu_baseline"] = cb
    else:
        line = run_struct(args, rank, world, dev)
        if rank == 0 and world == 1 and not args.no_cpu_baseline:
            line["cpu_baseline"] = (run_oracle_sample(args) if args.path == "structured"
                                    else run_oracle_spectral(args))
    if rank == 0:
        print(json.dumps(line))
    if world > 1:
        torch.distributed.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
