"""Busy-SM accounting of a CUPTI trace step (scripts/cupti_trace.cpp): per kernel
kind, sum of min(grid, 148) x duration, against 148 x step span."""
import csv
import re
import subprocess
import sys
from collections import defaultdict

rows = []
for r in csv.reader(open(sys.argv[1])):
    if len(r) >= 6:
        rows.append((int(r[0]), int(r[1]), int(r[2]), int(r[3]), int(r[4]), ",".join(r[5:])))
rows.sort()
g = [i for i, r in enumerate(rows) if "gather_kernel" in r[5]]
which = int(sys.argv[2]) if len(sys.argv) > 2 else -2
lo, hi = g[which], (g[which + 1] if which + 1 < 0 else len(rows))
dm = {}


def short(n):
    if n not in dm:
        d = subprocess.run(["c++filt", n], capture_output=True, text=True).stdout.strip()
        d = d.replace("(anonymous namespace)::", "").replace("pnb::", "").replace("void ", "")
        d = re.sub(r"\(.*", "", d)
        m = re.match(r"gemm_tc_kernel<(.*)>", d)
        dm[n] = ("gemm<" + m.group(1).replace("__nv_bfloat16", "bf16").replace("(bool)", "").replace("(int)", "") + ">") if m else d[:40]
    return dm[n]


t0 = rows[lo][0]
span = max(r[1] for r in rows[lo:hi]) - t0
acc = defaultdict(float)
for r in rows[lo:hi]:
    acc[short(r[5])] += min(r[4], 148) * (r[1] - r[0]) / 1e3
tot = sum(acc.values())
print(f"span {span / 1e3:.1f} us, busy SM-us {tot:.0f} = {tot / 148:.1f} us of the whole GPU ({tot / 148 / (span / 1e3) * 100:.0f}%)")
for k, v in sorted(acc.items(), key=lambda x: -x[1]):
    print(f"  {v / 148:7.1f} us  {k}")
