"""Per-kernel-kind GPU time of one kron-full NG step from a CUPTI trace
(trace_step.py ngsgd): sum of durations (serial view) and busy-SM time."""
import csv
import re
import subprocess
import sys
from collections import defaultdict

rows = sorted((int(r[0]), int(r[1]), int(r[4]), ",".join(r[5:])) for r in csv.reader(open(sys.argv[1])) if len(r) >= 6)
dm = {}


def short(n):
    if n not in dm:
        d = subprocess.run(["c++filt", n], capture_output=True, text=True).stdout.strip()
        d = d.replace("(anonymous namespace)::", "").replace("pnb::", "").replace("void ", "")
        d = re.sub(r"\(.*", "", d)
        dm[n] = d[:80]
    return dm[n]


g = [i for i, r in enumerate(rows) if "gather_kernel" in r[3]]
lo, hi = g[-2], g[-1]
span = rows[hi][0] - rows[lo][0]
dur, busy, cnt = defaultdict(float), defaultdict(float), defaultdict(int)
for r in rows[lo:hi]:
    k = short(r[3])
    dur[k] += (r[1] - r[0]) / 1e3
    busy[k] += min(r[2], 148) * (r[1] - r[0]) / 1e3 / 148
    cnt[k] += 1
print(f"step span {span / 1e3:.1f} us, {hi - lo} kernels, sum of durations {sum(dur.values()):.0f} us")
for k, v in sorted(dur.items(), key=lambda x: -x[1])[:25]:
    print(f"  {v:8.1f} us  x{cnt[k]:4d}  busy {busy[k]:7.1f} us  {k}")
