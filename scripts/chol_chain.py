"""Per-stream view of the kron-full NG factorizations in a CUPTI trace step:
streams with chol_diag launches, their busy time and gaps, and for the longest
chain the time by kernel kind plus the idle gaps before each kind."""
import csv
import re
import subprocess
import sys
from collections import defaultdict

rows = sorted((int(r[0]), int(r[1]), int(r[2]), int(r[4]), ",".join(r[5:])) for r in csv.reader(open(sys.argv[1]))
              if len(r) >= 6)
g = [i for i, r in enumerate(rows) if "gather_kernel" in r[4]]
lo, hi = g[-2], g[-1]
step = rows[lo:hi]
t0 = step[0][0]
dm = {}


def short(n):
    if n not in dm:
        d = subprocess.run(["c++filt", n], capture_output=True, text=True).stdout.strip()
        d = d.replace("(anonymous namespace)::", "").replace("pnb::", "").replace("void ", "")
        dm[n] = re.sub(r"\(.*", "", d)[:70]
    return dm[n]


by = defaultdict(list)
for r in step:
    by[r[2]].append(r)
print(f"step span {(rows[hi][0] - t0) / 1e3:.1f} us")
for sid, rs in sorted(by.items(), key=lambda x: -sum(1 for r in x[1] if "chol_diag" in r[4])):
    nd = sum(1 for r in rs if "chol_diag" in r[4])
    if nd == 0:
        continue
    busy = sum(r[1] - r[0] for r in rs)
    print(f"stream {sid}: {len(rs)} kernels, {nd} diag, busy {busy / 1e3:.1f} us, "
          f"{(rs[0][0] - t0) / 1e3:.1f} .. {(max(r[1] for r in rs) - t0) / 1e3:.1f} us")
sid = max(by, key=lambda s: sum(1 for r in by[s] if "chol_diag" in r[4]))
kinds = defaultdict(lambda: [0, 0.0, 0.0])
prev = None
for r in by[sid]:
    k = kinds[short(r[4])]
    k[0] += 1
    k[1] += (r[1] - r[0]) / 1e3
    if prev is not None:
        k[2] += max(0, r[0] - prev) / 1e3
    prev = r[1]
print(f"stream {sid} (most diag blocks): kind, count, busy us, idle-before us")
for n, (c, b, gp) in sorted(kinds.items(), key=lambda x: -x[1][1] - x[1][2]):
    print(f"  {c:4d} {b:9.1f} {gp:9.1f}  {n}")
