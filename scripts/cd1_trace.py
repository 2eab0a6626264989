"""Warm per-kernel durations of greedy_pretrain CD-1 steps from a CUPTI trace.

    LD_PRELOAD=scripts/libcupti_trace.so CUPTI_TRACE_OUT=gpurun_out/cd1.csv \
        python scripts/cd1_trace.py run [precision]
    python scripts/cd1_trace.py sum gpurun_out/cd1.csv

`run`: greedy_pretrain 2048-2048-2048-10 on 16384 frames x 2 epochs (256 CD-1
steps per RBM). `sum`: per kernel, median duration over the CD-1 steps, and the
median step span (load_rows start to the next load_rows start)."""
import csv
import os
import re
import statistics
import subprocess
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def run(prec):
    from paper_1507_01239_b200 import parnn as P
    x = np.random.default_rng(0).standard_normal((16384, 2048))
    ctx = P.Context(0)
    P.greedy_pretrain([2048, 2048, 2048, 10], x, P.PretrainOptions(2), seed=2, precision=P.Precision[prec], ctx=ctx)


def short(n):
    d = subprocess.run(["c++filt", n], capture_output=True, text=True).stdout.strip()
    d = d.replace("(anonymous namespace)::", "").replace("pnb::", "").replace("void ", "")
    return re.sub(r"\(.*", "", d)[:60]


def summarize(path):
    rows = sorted((int(r[0]), int(r[1]), ",".join(r[5:])) for r in csv.reader(open(path)) if len(r) >= 6)
    names = {n: short(n) for n in {r[2] for r in rows}}
    starts = [i for i, r in enumerate(rows) if "load_rows" in names[r[2]]]
    spans, per = [], {}
    for a, b in zip(starts, starts[1:]):
        if b - a != 9:  # a CD-1 step: load_rows + 4 GEMMs + 3 reductions + bias_finish
            continue
        spans.append(rows[b][0] - rows[a][0])
        for i in range(a, b):
            per.setdefault((i - a, names[rows[i][2]]), []).append(rows[i][1] - rows[i][0])
    print(f"{len(spans)} CD-1 steps, median span {statistics.median(spans) / 1e3:.1f} us")
    tot = 0.0
    for (k, n), d in sorted(per.items()):
        m = statistics.median(d) / 1e3
        tot += m
        print(f"  {k} {m:7.2f} us  {n}")
    print(f"  sum of kernel medians {tot:.1f} us")


if __name__ == "__main__":
    if sys.argv[1] == "run":
        run(sys.argv[2] if len(sys.argv) > 2 else "tf32")
    else:
        summarize(sys.argv[2])
