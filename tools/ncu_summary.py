"""Markdown rows (the columns of profiles/r01/ncu_fkernels_summary.md) from ncu --set full reports.
Usage: python tools/ncu_summary.py "label=path.ncu-rep" ..."""
import csv
import io
import subprocess
import sys

COLS = [("gpu__time_duration.sum", "time"), ("sm__inst_issued.avg.pct_of_peak_sustained_active", "issue %"),
        ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "FP64 pipe %"),
        ("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "XU %"),
        ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM %"),
        ("lts__t_sectors_srcunit_tex_op_read.sum", "L2 read sectors"),
        ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
        ("launch__registers_per_thread", "regs"), ("launch__cluster_max_active", "max clusters")]
STALL = "smsp__pcsamp_warps_issue_stalled_"


def row(label, path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, u, v = rows[0], rows[1], rows[2]
    get = {name: (v[i], u[i]) for i, name in enumerate(h)}
    cells = []
    for m, _ in COLS:
        val, unit = get.get(m, ("-", ""))
        if m == "gpu__time_duration.sum" and val != "-":
            x = float(val.replace(",", ""))
            x = x / 1e3 if unit == "ns" else (x * 1e3 if unit == "ms" else x)
            cells.append(f"{x:.1f} us" if x < 1000 else f"{x / 1e3:.2f} ms")
        else:
            cells.append(val)
    st = {k[len(STALL):]: float(val.replace(",", "") or 0) for k, (val, _) in get.items()
          if k.startswith(STALL) and not k.endswith("not_issued") and val not in ("", "-")}
    tot = sum(st.values()) or 1.0
    top = ", ".join(f"{k} {100 * x / tot:.0f}%" for k, x in sorted(st.items(), key=lambda t: -t[1])[:3])
    return f"| {label} | " + " | ".join(cells) + f" | {top} |"


if __name__ == "__main__":
    print("| kernel / workload | " + " | ".join(c for _, c in COLS) + " | top stalls |")
    print("|---" * (len(COLS) + 2) + "|")
    for arg in sys.argv[1:]:
        label, path = arg.rsplit("=", 1)
        print(row(label, path))
