"""Per-step GPU vs oracle low-rank state for a given (period, lag), fp32."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import ng_lowrank as LR  # noqa: E402
from oracle import parnn_oracle as O  # noqa: E402
from paper_1507_01239_b200 import parnn as P  # noqa: E402

period, lag = int(sys.argv[1]), int(sys.argv[2])
x, y = O.generate_synthetic(12, 40, 40, 4.0, 1)
mean, sd = O.feature_stats(x)
x = O.standardize(x, mean, sd)
dims = [40, 48, 36, 12]
B = 32
perm = np.random.default_rng(0).permutation(x.shape[0])
batches = [perm[(i * B + np.arange(B)) % x.shape[0]] for i in range(8)]
lrs = np.full(8, 0.3, np.float32)
cfg = LR.LowRankConfig(rank_in=6, rank_out=8, update_period=period, init_iters=3, update_lag=lag)
ctx = P.Context(0)
ds = P.DeviceDataset(ctx, P.Dataset(x, y.astype(np.int32), 12))
m = P.init_random(dims, seed=3)
r = P.Replica(ctx, dims, precision=P.Precision.fp32, optimizer=P.OptimizerKind.ngsgd_lowrank, minibatch=B, max_steps=8)
r.set_lowrank(6, 8, period, 3, 2000.0, lag)
r.set_params(m.params)
r.bind(ds)
r.upload_epoch(np.concatenate(batches), lrs)
om = O.unflatten(m.params, dims)
st = LR.lowrank_init(om, cfg)
for t in range(8):
    r.step(1)
    r.sync()
    LR.lowrank_train_steps(om, st, x, y, [batches[t]], [0.3])
    errs = []
    for l in range(3):
        for side, so in ((0, st.sides_in[l]), (1, st.sides_out[l])):
            w, d, rho = r.lowrank_state(l, side)
            dg = r.lowrank_diag(l, side)
            errs.append((l, side, round(abs(rho - so.rho) / so.rho, 6), round(float(np.abs(d - so.d).max() / so.d.max()), 6),
                         round(dg["trxx"], 4)))
    print(t, "params rel", np.linalg.norm(r.get_params() - O.flatten(om)) / np.linalg.norm(O.flatten(om)), errs[4:])
