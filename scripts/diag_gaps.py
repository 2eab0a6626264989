"""Start-to-start gaps of the output factor's diagonal blocks in a traced kron step
(the 8806 factor's 69 blocks are the diag launches that run last)."""
import csv
import sys

rows = sorted((int(r[0]), int(r[1]), ",".join(r[5:])) for r in csv.reader(open(sys.argv[1])) if len(r) >= 6)
g = [i for i, r in enumerate(rows) if "gather_kernel" in r[2]]
lo, hi = g[-2], g[-1]
t0 = rows[lo][0]
diag = [(r[0] - t0, r[1] - r[0]) for r in rows[lo:hi] if "chol_diag" in r[2]]
tail = diag[-69:]
gaps = [b[0] - a[0] for a, b in zip(tail, tail[1:])]
print(f"last 69 diag launches: {tail[0][0] / 1e3:.1f} .. {(tail[-1][0] + tail[-1][1]) / 1e3:.1f} us")
for i in range(0, 68, 4):
    seg = gaps[i:i + 4]
    print(f"  blocks {i:2d}-{i + 3:2d}: gaps {' '.join(f'{x / 1e3:6.1f}' for x in seg)} us; diag dur "
          f"{' '.join(f'{d / 1e3:5.1f}' for _, d in tail[i:i + 4])}")
