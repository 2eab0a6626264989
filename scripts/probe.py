"""Quick GPU probe: forward / SGD / NG parity vs the numpy oracle and a timing."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_1507_01239_b200 import parnn as P
from oracle import parnn_oracle as O

def rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30))

ctx = P.Context(0)
dims = [40, 64, 48, 10]
tr, cv = P.make_data(10, 40, 30, 6.0, 1)
m0 = P.init_random(dims, seed=3)
om = O.unflatten(m0.params, dims)
ds = P.DeviceDataset(ctx, tr)
for prec in (P.Precision.tf32, P.Precision.bf16):
    B = 32
    rows = np.arange(4 * B) % tr.size()
    try:
        r = P.Replica(ctx, dims, precision=prec, optimizer=P.OptimizerKind.sgd, minibatch=B, max_steps=4)
        r.set_params(m0.params)
        r.bind(ds)
        z = r.forward(ds, rows[:B])
        oz = O.forward(om, tr.features[rows[:B]]).z[-1]
        print(prec.name, "forward rel", rel(z, oz), flush=True)
        lrs = [0.3, 0.2, 0.1, 0.05]
        r.upload_epoch(rows, lrs)
        r.step(4); r.sync()
        ce = r.ce(4)
        mm = om.copy(); oces = []
        for s in range(4):
            rr = rows[s*B:(s+1)*B]; t = O.forward(mm, tr.features[rr]); oces.append(O.cross_entropy(t, tr.labels[rr]))
            gW, gb = O.backward(mm, t, tr.labels[rr]); O.sgd_step(mm, gW, gb, lrs[s])
        p = r.get_params(); op = O.flatten(mm)
        print(prec.name, "sgd ce", ce, oces, "theta rel", rel(p, op), "dtheta rel", rel(p - m0.params, op - m0.params), flush=True)
        # NG
        rn = P.Replica(ctx, dims, precision=prec, optimizer=P.OptimizerKind.ngsgd, minibatch=B, max_steps=4)
        rn.set_params(m0.params); rn.bind(ds); rn.upload_epoch(rows, lrs); rn.step(4); rn.sync()
        mm = om.copy(); st = O.ng_init(mm)
        for s in range(4):
            rr = rows[s*B:(s+1)*B]; t = O.forward(mm, tr.features[rr])
            gW, gb, dzs = O.backward(mm, t, tr.labels[rr], True); O.ng_update_state(st, t, dzs)
            gW, gb = O.ng_precondition(st, gW, gb); O.sgd_step(mm, gW, gb, lrs[s])
        p = rn.get_params(); op = O.flatten(mm)
        f = rn.get_ng_state()
        print(prec.name, "ng theta rel", rel(p, op), "dtheta rel", rel(p - m0.params, op - m0.params),
              "r_in0 rel", rel(f[0][0], st.r_in[0]), "r_out2 rel", rel(f[2][1], st.r_out[2]), flush=True)
        print("kernels/step sgd", r.kernels_per_step(), "ng", rn.kernels_per_step(), flush=True)
    except Exception as e:
        import traceback; traceback.print_exc()

# timing config 2 SGD bf16
dims2 = [440] + [2048] * 6 + [8806]
B = 1024
n = 16384
x = np.random.default_rng(0).standard_normal((n, 440))
y = np.random.default_rng(1).integers(0, 8806, n).astype(np.int32)
big = P.DeviceDataset(ctx, P.Dataset(x, y, 8806))
m2 = P.init_random(dims2, seed=1)
for prec in (P.Precision.bf16, P.Precision.tf32):
    for opt in (P.OptimizerKind.sgd, P.OptimizerKind.ngsgd):
        steps = 8 if opt == P.OptimizerKind.sgd else 3
        r = P.Replica(ctx, dims2, precision=prec, optimizer=opt, minibatch=B, max_steps=steps)
        r.set_params(m2.params); r.bind(big)
        rows = np.random.default_rng(2).integers(0, n, steps * B)
        r.upload_epoch(rows, [1e-3] * steps)
        r.step(1); r.sync()
        r.upload_epoch(rows, [1e-3] * steps)
        t0 = time.time(); r.step(steps); r.sync(); dt = (time.time() - t0) / steps
        print(f"cfg2 {prec.name} {opt.name}: {dt*1e3:.3f} ms/step, {B/dt:.0f} frames/s, CE {r.ce(steps)[:3]}", flush=True)
        r.close()
