"""GPU low-rank NG state vs the oracle, step by step, on mean-dominated
(sigmoid-like) inputs. Debug aid."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import ng_lowrank as LR  # noqa: E402
from oracle import parnn_oracle as O  # noqa: E402
from paper_1507_01239_b200 import parnn as P  # noqa: E402

dx = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
prec = sys.argv[2] if len(sys.argv) > 2 else "fp32"
rin = int(sys.argv[3]) if len(sys.argv) > 3 else 20
dims = [dx, 64, 16]
B = 1024
rng = np.random.default_rng(0)
n = 4096
z = rng.standard_normal((n, dx)) * 1.5 + rng.standard_normal(dx)
x = 1 / (1 + np.exp(-z))
y = (np.arange(n) % 16).astype(np.int32)
steps = 6
batches = [np.arange(i * B, (i + 1) * B) % n for i in range(steps)]
lrs = np.full(steps, 0.05, np.float32)
cfg = LR.LowRankConfig(rank_in=rin, rank_out=8, update_period=2, init_iters=3)
ctx = P.Context(0)
ds = P.DeviceDataset(ctx, P.Dataset(x, y, 16))
m = P.init_random(dims, seed=3)
r = P.Replica(ctx, dims, precision=P.Precision[prec], optimizer=P.OptimizerKind.ngsgd_lowrank, minibatch=B,
              max_steps=steps)
r.set_lowrank(cfg.rank_in, cfg.rank_out, cfg.update_period, cfg.init_iters, cfg.num_samples_history, cfg.update_lag)
r.set_params(m.params)
r.bind(ds)
r.upload_epoch(np.concatenate(batches), lrs)
om = O.unflatten(m.params, dims)
st = LR.lowrank_init(om, cfg)
for t in range(steps):
    r.step(1)
    r.sync()
    LR.lowrank_train_steps(om, st, x, y, [batches[t]], [float(lrs[t])])
    for l in range(2):
        for side, so in ((0, st.sides_in[l]), (1, st.sides_out[l])):
            w, d, rho = r.lowrank_state(l, side)
            print(f"t={t} l={l} s={side} gpu d0={d[0]:.4e} d1={d[1]:.4e} rho={rho:.4e} | ora d0={so.d[0]:.4e} "
                  f"d1={so.d[1]:.4e} rho={so.rho:.4e} | proj rel {np.linalg.norm(w.T@w - so.W.T@so.W)/np.linalg.norm(so.W.T@so.W):.2e}")
    p = r.get_params()
    print("   params rel", np.linalg.norm(p - O.flatten(om)) / np.linalg.norm(O.flatten(om)), flush=True)
