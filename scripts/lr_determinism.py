"""Two identical config-2 low-rank replicas stepped side by side must stay
bitwise equal (race detector for the concurrent step)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1507_01239_b200 import parnn as P  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 24
dims = [440] + [2048] * 6 + [8806]
rng = np.random.default_rng(0)
n = 4096
x = rng.standard_normal((n, 440))
y = (np.arange(n) % 8806).astype(np.int32)
ctx = P.Context(0)
ds = P.DeviceDataset(ctx, P.Dataset(x, y, 8806))
reps = []
for _ in range(2):
    r = P.Replica(ctx, dims, precision=P.Precision.bf16, optimizer=P.OptimizerKind.ngsgd_lowrank, minibatch=1024,
                  max_steps=steps + 4)
    r.set_params(P.init_random(dims, seed=1).params)
    r.bind(ds)
    r.upload_epoch(np.resize(np.arange(n), (steps + 4) * 1024), np.full(steps + 4, 1e-3, np.float32))
    reps.append(r)
for t in range(steps):
    for r in reps:
        r.step(1)
    errs = []
    for r in reps:
        try:
            r.sync()
            errs.append(None)
        except Exception as e:
            errs.append(str(e))
    p0, p1 = reps[0].get_params(), reps[1].get_params()
    same = np.array_equal(p0, p1)
    print(t, "equal", same, "finite", bool(np.all(np.isfinite(p0))), bool(np.all(np.isfinite(p1))), errs, flush=True)
    if not same or any(errs):
        d = np.abs(p0 - p1)
        print("  maxdiff", np.nanmax(d), "first idx", int(np.argmax(d > 0)))
        break
