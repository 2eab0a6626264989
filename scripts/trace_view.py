"""Summarise a CUPTI kernel trace (scripts/cupti_trace.cpp) of the low-rank step:
per step (split at gather kernels) the kernels sorted by start, with stream."""
import csv
import re
import sys

import subprocess

rows = []
for r in csv.reader(open(sys.argv[1])):
    if len(r) < 6:
        continue
    rows.append((int(r[0]), int(r[1]), int(r[2]), int(r[3]), int(r[4]), ",".join(r[5:])))
rows.sort()
gathers = [i for i, r in enumerate(rows) if "gather_kernel" in r[5]]
which = int(sys.argv[2]) if len(sys.argv) > 2 else -3
lo = gathers[which]
hi = gathers[which + 1] if which + 1 < len(gathers) and which != -1 else len(rows)
t0 = rows[lo][0]


_dm = {}


def demangle(n):
    if n not in _dm:
        _dm[n] = subprocess.run(["c++filt", n], capture_output=True, text=True).stdout.strip()
    return _dm[n]


def short(n):
    n = demangle(n).replace("(anonymous namespace)::", "")
    n = re.sub(r"\(.*", "", n)
    n = n.replace("void ", "").replace("pnb::", "").replace("(anonymous namespace)::", "")
    m = re.match(r"gemm_tc_kernel<(.*)>", n)
    if m:
        return "gemm<" + m.group(1).replace("__nv_bfloat16", "bf16").replace("(bool)", "").replace("(int)", "") + ">"
    return n[:40]


streams = {}
for r in rows[lo:hi]:
    streams.setdefault(r[2], len(streams))
end = max(r[1] for r in rows[lo:hi])
print(f"step {which}: {(end - t0) / 1e3:.1f} us, {hi - lo} kernels, {len(streams)} streams")
for r in rows[lo:hi]:
    print(f"{(r[0] - t0) / 1e3:8.1f} {(r[1] - t0) / 1e3:8.1f} {(r[1] - r[0]) / 1e3:7.1f}  s{streams[r[2]]:<2d} grid {r[4]:4d}  {short(r[5])}")
