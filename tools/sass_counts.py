"""Static SASS instruction counts of the hot kernels in libsplidar.so (cuobjdump -sass), for
profiles/: proves which units a kernel uses (UTCIMMA = tcgen05.mma kind::i8 on the 5th-gen tensor
cores, LDTM = tcgen05.ld TMEM -> registers, UTMALDG = tensor-map TMA, UBLKCP = 1-D bulk TMA,
DMMA = FP64 tensor cores, SYNCS = mbarrier ops). python tools/sass_counts.py > profiles/r02/sass_counts.md"""
import collections
import re
import subprocess
import sys
import os

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2509_20500_b200", "lib", "libsplidar.so")
OPS = ["UTCIMMA", "LDTM", "UTCBAR", "UTMALDG", "UBLKCP", "DMMA", "DFMA", "DADD", "DMUL", "SYNCS", "PRMT",
       "LDS", "STS", "LDG", "STG", "SHFL", "BAR", "MUFU", "F2F"]
WANT = ["k_power_step_i8IfE", "k_power_step_i8e", "k_enc_colexp", "k_power_step_i8IdE", "k_power_stepIdLi17E", "k_power_stepIfLi17E", "k_power_stepIdLi1E",
        "k_power_check", "k_power_loopIdLi17E", "k_power_loopIdLi1E", "k_i8_colexpIfE", "k_buildIdLi0E", "k_power_fusedIdLi1E", "k_struct_solve_c1", "k_mc"]

sass = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True).stdout
funcs = re.split(r"\n\s*Function : ", sass)
rows = []
for f in funcs[1:]:
    name = f.split("\n", 1)[0].strip()
    if not any(w in name for w in WANT):
        continue
    cnt = collections.Counter()
    for line in f.splitlines():
        m = re.match(r"\s+/\*[0-9a-f]{4,}\*/\s+(@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)", line)
        if m:
            cnt[m.group(2)] += 1
    total = sum(cnt.values())
    short = next(w for w in WANT if w in name)
    rows.append((short, total, cnt))
print("| kernel (mangled stem) | SASS instr | " + " | ".join(OPS) + " |")
print("|---" * (len(OPS) + 2) + "|")
for short, total, cnt in rows:
    print(f"| {short} | {total} | " + " | ".join(str(cnt.get(o, 0)) for o in OPS) + " |")
