"""Run a few config-2 low-rank NG-SGD steps (for ncu launch lists / timelines).

    python scripts/lr_steps.py [--steps N] [--warmup W] [--precision bf16] [--optimizer ngsgd_lowrank]
"""
import argparse
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1507_01239_b200 import parnn as P  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--steps", type=int, default=4)
ap.add_argument("--warmup", type=int, default=5)
ap.add_argument("--precision", default="bf16")
ap.add_argument("--optimizer", default="ngsgd_lowrank")
ap.add_argument("--time", action="store_true")
ap.add_argument("--bench-data", action="store_true", help="bench.py's generate_synthetic data (8806 x 24)")
a = ap.parse_args()
dims = [440] + [2048] * 6 + [8806]
rng = np.random.default_rng(0)
ctx = P.Context(0)
if a.bench_data:
    train, _ = P.make_data(8806, 440, 24, 8.0, 1, 0.10, 2, True)
    x, y = train.features, train.labels
    n = x.shape[0]
else:
    n = 4096
    x = rng.standard_normal((n, 440))
    y = (np.arange(n) % 8806).astype(np.int32)
ds = P.DeviceDataset(ctx, P.Dataset(x, y, 8806))
r = P.Replica(ctx, dims, precision=P.Precision[a.precision], optimizer=P.OptimizerKind[a.optimizer], minibatch=1024,
              max_steps=a.steps + a.warmup + 128)
r.set_params(P.init_random(dims, seed=1).params)
if os.environ.get("LR_LAG") or os.environ.get("LR_RANK_OUT"):
    r.set_lowrank(update_lag=int(os.environ.get("LR_LAG", 4)), rank_out=int(os.environ.get("LR_RANK_OUT", 80)))
r.bind(ds)
tot = a.steps + a.warmup + 128
r.upload_epoch(np.resize(np.arange(n), tot * 1024), np.full(tot, 1e-3, np.float32))
r.step(a.warmup)
r.sync()
if a.time:
    ms = r.time_steps(40) / 40
    print(f"ms/step {ms:.4f}  frames/s {1024 / ms * 1e3:.0f}  kernels/step {r.kernels_per_step()}")
else:
    r.step(a.steps)
    r.sync()
print("ce", r.ce(a.warmup + (40 if a.time else a.steps))[-3:])
if os.environ.get("LR_PROFILE"):
    for rep in range(2):
        prof = r.profile(2)
        print("profile", rep, [(n, round(t, 4)) for n, t, f in prof][:12])

if os.environ.get("LR_EIGTIME"):
    r.step(3)
    r.sync()
    rows = []
    for l in range(len(dims) - 1):
        for side in (0, 1):
            d = r.lowrank_diag(l, side)
            rows.append((d["eig_start_ns"], d["eig_end_ns"], l, side, d["sweeps"]))
    t0 = min(x[0] for x in rows)
    for e0, e1, l, side, sw in sorted(rows):
        print(f"layer {l} {'in ' if side == 0 else 'out'} eig {((e0 - t0) / 1e3):8.1f} .. {((e1 - t0) / 1e3):8.1f} us  sweeps {sw}")
if os.environ.get("LR_PERSTEP"):
    import collections
    acc = collections.defaultdict(list)
    for i in range(40):
        t = a.warmup + 40 + i if a.time else a.warmup + a.steps + i
        acc[i % 4].append(r.time_steps(1))
    print("per-step ms by phase in the update period:", {k: round(sum(v) / len(v), 4) for k, v in sorted(acc.items())})
