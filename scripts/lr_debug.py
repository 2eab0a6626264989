"""Step a config-2 low-rank replica one step at a time and report the first
non-finite NG state / parameters, plus Jacobi sweep diagnostics."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1507_01239_b200 import parnn as P  # noqa: E402

dims = [440] + [2048] * 6 + [8806]
rng = np.random.default_rng(0)
n = 4096
x = rng.standard_normal((n, 440))
y = (np.arange(n) % 8806).astype(np.int32)
ctx = P.Context(0)
ds = P.DeviceDataset(ctx, P.Dataset(x, y, 8806))
steps = int(sys.argv[1]) if len(sys.argv) > 1 else 40
r = P.Replica(ctx, dims, precision=P.Precision.bf16, optimizer=P.OptimizerKind.ngsgd_lowrank, minibatch=1024,
              max_steps=steps + 4)
r.set_params(P.init_random(dims, seed=1).params)
r.bind(ds)
r.upload_epoch(np.resize(np.arange(n), (steps + 4) * 1024), np.full(steps + 4, 1e-3, np.float32))
for t in range(steps):
    r.step(1)
    try:
        r.sync()
    except Exception as e:
        print("step", t, "error", e)
        for l in range(len(dims) - 1):
            for side in (0, 1):
                w, d, rho = r.lowrank_state(l, side)
                dg = r.lowrank_diag(l, side)
                print(f"  l={l} side={side} finite={np.all(np.isfinite(w))} rho={rho:.3e} d[:2]={d[:2]} d[-1]={d[-1]:.3e} "
                      f"|w|={np.abs(w).max():.3e} trxx={dg['trxx']:.3e} gamma={dg['gamma']:.3e} sweeps={dg['sweeps']} "
                      f"cyc={dg['jacobi_cycles']:.3e}")
        p = r.get_params()
        print("params finite", np.all(np.isfinite(p)), "max", np.abs(p).max())
        break
    bad = []
    for l in range(len(dims) - 1):
        for side in (0, 1):
            w, d, rho = r.lowrank_state(l, side)
            if not (np.all(np.isfinite(w)) and np.all(np.isfinite(d)) and np.isfinite(rho)):
                bad.append((l, side))
            dg = r.lowrank_diag(l, side)
            if t in (0, 1, 4, 5, 9, 16, 19, 20) and l in (0, 3, 4, 6):
                print(f"t={t} l={l} side={side} rho={rho:.3e} d[:2]={d[:2]} d[-1]={d[-1]:.3e} |w|={np.abs(w).max():.3e}"
                      f" trxx={dg['trxx']:.3e} gamma={dg['gamma']:.3e} sweeps={dg['sweeps']} cyc={dg['jacobi_cycles']:.3e}")
    p = r.get_params()
    print(t, "ce", r.ce(t + 1)[-1], "params finite", bool(np.all(np.isfinite(p))), "bad sides", bad[:6], flush=True)
    if bad:
        break
