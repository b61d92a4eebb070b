"""Summarise one kernel of an ncu report: headline metrics, stall reasons and the hottest SASS lines.

python tools/ncu_top.py REPORT.ncu-rep KERNEL_REGEX [N_LINES]
"""
import csv
import io
import subprocess
import sys

rep, kre = sys.argv[1], sys.argv[2]
nl = int(sys.argv[3]) if len(sys.argv) > 3 else 15


def ncu(*args):
    return subprocess.run(["ncu", "-i", rep, "-k", f"regex:{kre}", *args], capture_output=True, text=True).stdout


r = list(csv.reader(io.StringIO(ncu("--page", "details", "--csv"))))
h = r[0]
mi, vi, ui = h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit")
want = ["Duration", "SM Frequency", "DRAM Throughput", "Memory Throughput", "Compute (SM) Throughput",
        "Executed Ipc Active", "Issue Slots Busy", "No Eligible", "Registers Per Thread"]
for row in r[1:]:
    if row[mi] in want:
        print(f"{row[mi]:28s} {row[vi]} {row[ui]}")
raw = list(csv.reader(io.StringIO(ncu("--page", "raw", "--csv"))))
h, v = raw[0], raw[2]
st = []
for i, name in enumerate(h):
    if "smsp__pcsamp_warps_issue_stalled" in name and not name.endswith("not_issued"):
        try:
            st.append((float(v[i].replace(",", "")), name.replace("smsp__pcsamp_warps_issue_stalled_", "")))
        except ValueError:
            pass
tot = sum(x for x, _ in st) or 1
print("stalls:", ", ".join(f"{n} {x / tot * 100:.0f}%" for x, n in sorted(st, reverse=True)[:8]))
src = list(csv.reader(io.StringIO(ncu("--page", "source", "--csv", "--print-source", "sass"))))
h = src[1]
ai, si, wi = h.index("Address"), h.index("Source"), h.index("Warp Stall Sampling (All Samples)")
seen, data = set(), []
for i, row in enumerate(src[2:]):
    if row[ai] in seen:
        continue
    seen.add(row[ai])
    try:
        data.append((float(row[wi] or 0), len(data), row[si]))
    except ValueError:
        pass
tot = sum(d[0] for d in data) or 1
for x, i, s in sorted(data, reverse=True)[:nl]:
    print(f"{x / tot * 100:5.1f}% #{i:5d} {s[:100]}")
