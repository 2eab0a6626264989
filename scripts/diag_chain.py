"""Chain view of the kron-full NG factorization in a CUPTI trace (trace_step.py ngsgd):
duration and spacing of the chol_diag launches of one step (the 8806 factor's chain is
the long tail). Usage: python scripts/diag_chain.py trace.csv"""
import csv
import sys

rows = sorted((int(r[0]), int(r[1]), ",".join(r[5:])) for r in csv.reader(open(sys.argv[1])) if len(r) >= 6)
g = [i for i, r in enumerate(rows) if "gather_kernel" in r[2]]
a, b = g[-2], g[-1]
step = rows[a:b]
t0 = step[0][0]
d = [r for r in step if "chol_diag" in r[2]]
last = d[-69:]
durs = [(r[1] - r[0]) / 1e3 for r in last]
gaps = [(last[i][0] - last[i - 1][1]) / 1e3 for i in range(1, len(last))]
print(f"step {(rows[b][0] - t0) / 1e3:.1f} us; {len(d)} diag launches")
print(f"last 69 diag: {(last[0][0] - t0) / 1e3:.1f} .. {(last[-1][1] - t0) / 1e3:.1f} us")
print(f"  duration mean {sum(durs) / len(durs):.1f} min {min(durs):.1f} max {max(durs):.1f} us")
print(f"  start-to-start mean {((last[-1][0] - last[0][0]) / 1e3) / (len(last) - 1):.1f} us, gap after diag mean {sum(gaps) / len(gaps):.1f} us")
