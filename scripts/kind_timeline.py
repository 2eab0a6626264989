"""First start / last end / count / summed duration per kernel kind in one traced step.

    python scripts/kind_timeline.py trace.csv [k]   (k: the k-th last complete step, default 1)"""
import csv
import re
import subprocess
import sys
from collections import defaultdict

rows = sorted((int(r[0]), int(r[1]), int(r[4]), ",".join(r[5:])) for r in csv.reader(open(sys.argv[1])) if len(r) >= 6)
g = [i for i, r in enumerate(rows) if "gather_kernel" in r[3]]
kb = int(sys.argv[2]) if len(sys.argv) > 2 else 1
lo, hi = g[-1 - kb], g[-kb]
step = rows[lo:hi]
t0 = step[0][0]
dm = {}


def short(n):
    if n not in dm:
        d = subprocess.run(["c++filt", n], capture_output=True, text=True).stdout.strip()
        d = d.replace("(anonymous namespace)::", "").replace("pnb::", "").replace("void ", "")
        dm[n] = re.sub(r"\(.*", "", d)[:72]
    return dm[n]


k = defaultdict(lambda: [1e18, 0, 0, 0.0])
for r in step:
    a = k[short(r[3])]
    a[0] = min(a[0], r[0] - t0)
    a[1] = max(a[1], r[1] - t0)
    a[2] += 1
    a[3] += (r[1] - r[0]) / 1e3
print(f"step span {(rows[hi][0] - t0) / 1e3:.1f} us")
for n, (s, e, c, d) in sorted(k.items(), key=lambda x: x[1][1]):
    print(f"  {s / 1e3:9.1f} .. {e / 1e3:9.1f} us  x{c:4d}  sum {d:8.1f} us  {n}")
