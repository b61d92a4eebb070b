"""Parses the ncu --metrics captures written by tools/gpu_bench_all.sh (gpurun_out/ncu_*_metrics_*.csv:
the program's JSON line followed by ncu's CSV rows) into profiles/traffic.json entries (per-launch DRAM
bytes, FP64 flops per unit, FP64 pipe %), so the bench lines that follow use counts from the same code."""
import csv, json, os, sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")
path = os.path.join(ROOT, "profiles", "traffic.json")
t = json.load(open(path))


def parse(fname, kernel):
    rows, line = [], None
    for raw in open(fname):
        if raw.startswith("{"):
            line = json.loads(raw)
            continue
        r = next(csv.reader([raw]), [])
        if len(r) > 14 and kernel in r[4]:
            rows.append(r)
    m = {r[12]: float(r[14].replace(",", "")) for r in rows}
    return m, line


def flops(m):
    return (2 * m["smsp__sass_thread_inst_executed_op_dfma_pred_on.sum"] + m["smsp__sass_thread_inst_executed_op_dadd_pred_on.sum"]
            + m["smsp__sass_thread_inst_executed_op_dmul_pred_on.sum"])


for w, n in (("c5", 32768), ("c3", 4096)):
    f = os.path.join(OUT, f"ncu_eq4_metrics_{w}.csv")
    if os.path.exists(f):
        m, _ = parse(f, "k_build_eq4")
        t[f"{w}_eq4_f64"] = {"fp64_flops_per_entry": round(flops(m) / n / n, 2),
                             "dram_bytes": m["dram__bytes_read.sum"] + m["dram__bytes_write.sum"],
                             "fp64_pipe_pct": m["sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active"],
                             "source": f"profiles/r01/ncu_eq4_metrics_{w}.csv (ncu --metrics, one launch)"}
for w in ("c1", "grid"):
    f = os.path.join(OUT, f"ncu_mc_metrics_{w}.csv")
    if os.path.exists(f):
        m, line = parse(f, "k_mc")
        t[f"{w}_mc_f64"] = {"fp64_flops_per_registration": round(flops(m) / line["registrations_per_step"], 1),
                            "dram_bytes": m["dram__bytes_read.sum"] + m["dram__bytes_write.sum"],
                            "fp64_pipe_pct": m["sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active"],
                            "source": f"profiles/r01/ncu_mc_metrics_{w}.csv (ncu --metrics, one launch; flops / "
                                      "counted registrations of that step)"}
json.dump(t, open(path, "w"), indent=1)
json.dump(t, open(os.path.join(OUT, "traffic.json"), "w"), indent=1)
print(json.dumps(t, indent=1))
