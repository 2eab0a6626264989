"""Config 1 (440-512-512-1000, 100k frames, minibatch 256, 1 worker, averaging
period 4, lr 2.0, 2 epochs) with the reference's kron-full NG-SGD (golden from
the compiled reference: tests/golden/golden_cfg1_ng.npz) beside this
framework's kron-full NG and low-rank NG-SGD at update lag 1 and 4."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1507_01239_b200 import parnn as P  # noqa: E402

g = np.load(os.path.join(ROOT, "tests/golden/golden_cfg1_ng.npz"))
print("reference kron-full NG (fp64):", [tuple(np.round(r[2:4], 4)) for r in g["met"]])
dims = [440, 512, 512, 1000]
tr, cv = P.make_data(1000, 440, 100, float(g["separation"]), 7, 0.1, 2, True)
m0 = P.init_random(dims, seed=1)
ctx = P.Context(0)
plan = P.ParallelPlan(1, 4, 256, 5)
runs = [("ngsgd", P.Precision.fp32, 1), ("ngsgd_lowrank", P.Precision.fp32, 1), ("ngsgd_lowrank", P.Precision.fp32, 4),
        ("ngsgd_lowrank", P.Precision.bf16, 1), ("ngsgd_lowrank", P.Precision.bf16, 4)]
for opt, prec, lag in runs:
    o = P.TrainOptions(optimizer=P.OptimizerKind[opt], lr_init=float(g["lr_init"]), epochs=int(g["epochs"]),
                       precision=prec, ng_update_lag=lag)
    res = P.train_parallel(plan, m0, tr, cv, o, ctx=ctx)
    print(f"{opt:14s} {prec.name:5s} lag {lag}:", [(round(m.train_ce, 4), round(m.cv_accuracy, 4)) for m in res.metrics],
          flush=True)
