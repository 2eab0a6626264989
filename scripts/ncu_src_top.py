"""Top CUDA source lines by warp-stall samples from
`ncu -i X.ncu-rep --page source --csv --print-source cuda,sass` output, with
their dominant stall reasons (ncu's per-line aggregate rows). Usage:
    python scripts/ncu_src_top.py gpurun_out/r2_ncu_src_0.csv [N]"""
import csv
import sys


def num(v):
    try:
        return float(v)
    except ValueError:
        return 0.0


path = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
rows = list(csv.reader(open(path)))
lines, cur_file, hdr = [], "", None
for r in rows:
    if len(r) == 2 and r[0] == "File Path":
        cur_file = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = {n: i for i, n in reversed(list(enumerate(r)))}
        stalls = [n for n in r if n.startswith("stall_") and "Not Issued" not in n]
        continue
    if hdr and len(r) >= len(hdr) and r[0] and r[2] == "-":
        s = num(r[hdr["Warp Stall Sampling (All Samples)"]])
        st = sorted(((num(r[hdr[n]]), n) for n in set(stalls)), reverse=True)[:3]
        lines.append((s, cur_file, r[0], r[1].strip(), st))
tot = sum(x[0] for x in lines)
lines.sort(key=lambda x: -x[0])
print(f"total samples {tot:.0f}")
for s, f, ln, src, st in lines[:top]:
    print(f"{100 * s / tot:5.1f}%  {f}:{ln:<5} {src[:70]:70s} " + " ".join(f"{n[6:]}={v:.0f}" for v, n in st if v > 0))
