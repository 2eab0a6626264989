"""Debug: config-4 2048x2048 CD-1, three steps as in tests/test_rbm.py, per-column errors."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
from oracle import parnn_oracle as O
from paper_1507_01239_b200 import parnn as P
import test_rbm as T

ctx = P.Context(0)
v, h, gauss = 2048, 2048, False
prec = P.Precision[sys.argv[1] if len(sys.argv) > 1 else "fp32"]
W, vb, hb, x, rng = T._cfg4_case(v, h, gauss, 7 + v)
hb = T._margin_hb(W, hb, x)
r = P.Rbm(ctx, v, h, gauss, batch=128, precision=prec)
r.set_params(np.concatenate([W.ravel(), vb, hb]))
state = O.Rbm(W.copy(), vb.copy(), hb.copy(), gauss)
for step, mode in enumerate(("threshold", "uniforms", "threshold", "threshold")):
    xs = x if step < 2 else T.f32(np.roll(x, 5 * step, axis=0))
    if mode == "threshold" and step:
        hbm = T._margin_hb(state.W, T.f32(state.hb), xs)
        state = O.Rbm(T.f32(state.W), T.f32(state.vb), hbm, gauss)
        r.set_params(np.concatenate([state.W.ravel(), state.vb, state.hb]))
    hp = r.hidden_probs(xs)
    print(step, "hidden_probs err", np.abs(hp - O.hidden_probs(state, xs)).max(), "min|z|", np.abs(xs @ state.W.T + state.hb).min())
    before = np.concatenate([state.W.ravel(), state.vb, state.hb])
    if mode == "uniforms":
        p = O.hidden_probs(state, xs)
        u = rng.random(p.shape)
        near = np.abs(u - p) < 1e-4
        u[near] = np.where(p[near] > 0.5, p[near] - 2e-4, p[near] + 2e-4)
        sampler = lambda q, u=u: (u < q).astype(float)
        r.cd1(xs, 0.1, sampling="uniforms", uniforms=u.ravel())
    else:
        sampler = O.threshold_half
        r.cd1(xs, 0.1, sampling="threshold")
    pos, hs, rec, neg = O.cd1_gibbs(state, xs, sampler)
    new = O.cd1_apply(state, xs, pos, rec, neg, 0.1)
    got = r.get_params()
    gW, gv, gh = T.unpack(got, v, h)
    dW = gW - new.W
    dh = gh - new.hb
    print(step, mode, "dW max", np.abs(dW).max(), "dW col-max argmax rows", np.argsort(-np.abs(dW).max(1))[:5],
          "dhb max", np.abs(dh).max(), "argmax", np.argsort(-np.abs(dh))[:5], "dvb max", np.abs(gv - new.vb).max(),
          "|dW ref| max", np.abs(new.W - state.W).max(), "hs on frac", hs.mean())
    state = O.Rbm(*[a.copy() for a in T.unpack(got, v, h)], gauss)
