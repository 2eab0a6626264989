import sys, numpy as np
sys.path.insert(0, '/root/repo')
from paper_1507_01239_b200 import parnn as P
dims = [440] + [2048] * 6 + [8806]
ctx = P.Context(0)
for opt in ("ngsgd_lowrank", "sgd"):
    outs = []
    for sep in (20.0, 24.0, 20.0):
        tr, cv = P.DeviceDataset.generate(ctx, 8806, 440, 16, sep, 1, 0.10, 2, True)
        m0 = P.init_random(dims, seed=7)
        o = P.TrainOptions(optimizer=P.OptimizerKind[opt], lr_init=10.0, epochs=2, precision=P.Precision.bf16)
        res = P.train_parallel(P.ParallelPlan(1, 4, 1024, 5), m0, None, None, o, ctx=ctx, device_data=(tr, cv))
        print(opt, sep, [round(float(m.train_ce), 4) for m in res.metrics], float(np.abs(res.model.params).sum()), flush=True)
