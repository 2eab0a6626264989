"""Steady-state step time of config 2 (graph launches, CUDA events, averaging every 4):
python scripts/step_time.py [optimizer] [steps] -- prints ms/step over `steps` steps after 40 warm-up."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1507_01239_b200 import parnn as P  # noqa: E402

opt = P.OptimizerKind[sys.argv[1] if len(sys.argv) > 1 else "ngsgd_lowrank"]
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 400
dims = [440] + [2048] * 6 + [8806]
ctx = P.Context(0)
tr, _ = P.DeviceDataset.generate(ctx, 8806, 440, 16, 20.0, 1, 0.10, 2, True)
r = P.Replica(ctx, dims, precision=P.Precision.bf16, optimizer=opt, minibatch=1024, max_steps=steps + 48)
r.set_params(P.init_random(dims, seed=7).params)
r.bind(tr)
r.upload_epoch(np.random.default_rng(2).integers(0, tr.n, (steps + 48) * 1024), np.full(steps + 48, 1.0))
P.run_steps([r], 40, 4)
r.sync()
ms = [P.run_steps([r], steps // 4, 4) / (steps // 4) for _ in range(4)]
print(f"{sys.argv[1] if len(sys.argv) > 1 else 'ngsgd_lowrank'} {np.median(ms):.4f} ms/step (4 x {steps // 4} steps: "
      + " ".join(f"{m:.4f}" for m in ms) + ")", flush=True)
