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
a = ap.parse_args()
dims = [440] + [2048] * 6 + [8806]
rng = np.random.default_rng(0)
n = 4096
x = rng.standard_normal((n, 440))
y = (np.arange(n) % 8806).astype(np.int32)
ctx = P.Context(0)
ds = P.DeviceDataset(ctx, P.Dataset(x, y, 8806))
r = P.Replica(ctx, dims, precision=P.Precision[a.precision], optimizer=P.OptimizerKind[a.optimizer], minibatch=1024,
              max_steps=a.steps + a.warmup + 64)
r.set_params(P.init_random(dims, seed=1).params)
r.bind(ds)
tot = a.steps + a.warmup + 64
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
