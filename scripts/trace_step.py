"""Run graph-launched config-2 steps for a kernel trace (LD_PRELOAD=scripts/libcupti_trace.so,
CUPTI_TRACE_OUT=...): 12 warm-up steps, then 8 steps. Usage: python scripts/trace_step.py [optimizer]"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1507_01239_b200 import parnn as P  # noqa: E402

opt = P.OptimizerKind[sys.argv[1] if len(sys.argv) > 1 else "ngsgd_lowrank"]
dims = [440] + [2048] * 6 + [8806]
ctx = P.Context(0)
x = np.random.default_rng(0).standard_normal((8192, 440))
y = np.random.default_rng(1).integers(0, 8806, 8192).astype(np.int32)
ds = P.DeviceDataset(ctx, P.Dataset(x, y, 8806))
r = P.Replica(ctx, dims, precision=P.Precision.bf16, optimizer=opt, minibatch=1024, max_steps=40)
r.set_params(P.init_random(dims, seed=7).params)
r.bind(ds)
r.upload_epoch(np.random.default_rng(2).integers(0, 8192, 40 * 1024), np.full(40, 1e-3))
P.run_steps([r], 12, 4)
r.sync()
ms = P.run_steps([r], 8, 4)
r.sync()
print(f"{ms / 8:.4f} ms/step", flush=True)
