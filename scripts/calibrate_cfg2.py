"""Pick the config-2 throughput workload (SURVEY §8d "Calibrate s"): device-generated
synthetic frames (8806 classes x per_class, 440-dim), 440-2048x6-8806, minibatch
1024, bf16; per-epoch CE and CV accuracy for a grid of separations / learning
rates / optimizers, optionally from a greedy-pretrained (RBM CD-1) stack.
Usage: python scripts/calibrate_cfg2.py per_class epochs seps lrs opts [pretrain_frames]
  e.g. python scripts/calibrate_cfg2.py 128 6 16 10,30 ngsgd_lowrank,sgd 100000"""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1507_01239_b200 import parnn as P  # noqa: E402

per_class = int(sys.argv[1])
epochs = int(sys.argv[2])
seps = [float(v) for v in sys.argv[3].split(",")]
lrs = [float(v) for v in sys.argv[4].split(",")]
opts_ = sys.argv[5].split(",")
pre = int(sys.argv[6]) if len(sys.argv) > 6 else 0
dims = [440] + [2048] * 6 + [8806]
ctx = P.Context(0)
for sep in seps:
    tr, cv = P.DeviceDataset.generate(ctx, 8806, 440, per_class, sep, 1, 0.10, 2, True)
    inits = {"random": P.init_random(dims, seed=7)}
    if pre:
        t0 = time.time()
        x = tr.download().features[np.random.default_rng(0).permutation(tr.n)[:pre]].astype(np.float64)
        inits["rbm"] = P.greedy_pretrain(dims, x, P.PretrainOptions(epochs=3), seed=7, precision=P.Precision.bf16,
                                         ctx=ctx)
        print(f"s={sep:g} pretrain {pre} frames x 3 epochs: {time.time() - t0:.1f}s", flush=True)
    for name, m0 in inits.items():
        for opt in opts_:
            for lr in lrs:
                o = P.TrainOptions(optimizer=P.OptimizerKind[opt], lr_init=lr, epochs=epochs, precision=P.Precision.bf16)
                t0 = time.time()
                res = P.train_parallel(P.ParallelPlan(1, 4, 1024, 5), m0, None, None, o, ctx=ctx,
                                       device_data=(tr, cv))
                print(f"s={sep:g} init={name} {opt} lr={lr:g} {time.time() - t0:.1f}s",
                      [(round(float(m.train_ce), 3), round(float(m.cv_accuracy), 4)) for m in res.metrics], flush=True)
