"""Kron-full NG trajectory vs the compiled reference on a small config-1 set
(tests/golden/_tmp_ref_ng_pc*.npz from the reference): final params and
epoch metrics, fp32 mode."""
import os, sys, glob
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1507_01239_b200 import parnn as P
dims = [440, 512, 512, 1000]
ctx = P.Context(0)
for f in sorted(glob.glob(os.path.join(ROOT, "tests/golden/_tmp_ref_ng_pc*.npz"))):
    pc = int(f.split("_pc")[1].split("_")[0]); ep = int(f.split("_ep")[1].split(".")[0])
    g = np.load(f)
    tr, cv = P.make_data(1000, 440, pc, 16.0, 7, 0.1, 2, True)
    m0 = P.init_random(dims, seed=1)
    for prec in (P.Precision.fp32, P.Precision.bf16):
        o = P.TrainOptions(optimizer=P.OptimizerKind.ngsgd, lr_init=2.0, epochs=ep, precision=prec)
        res = P.train_parallel(P.ParallelPlan(1, 4, 256, 5), m0, tr, cv, o, ctx=ctx)
        p = res.model.params
        print(os.path.basename(f), prec.name, "ref met", g["met"][:, [1, 2, 3, 6]].tolist(), "ours",
              [(m.lr, m.train_ce, m.cv_accuracy, m.avg_events) for m in res.metrics],
              "param rel err", np.linalg.norm(p - g["p"]) / np.linalg.norm(g["p"]),
              "delta rel err", np.linalg.norm(p - g["p"]) / np.linalg.norm(g["p"] - m0.params), flush=True)
