"""RBM CD-1 parity (pretrain.cpp:37-136).

The device CD-1 step -- three split-K GEMMs with fused reductions (sigmoid,
Bernoulli draw, reconstruction, column sums), the rank-2b weight update and the
bias update -- against the pinned numpy oracle (oracle/parnn_oracle.py
cd1_gibbs / cd1_apply, itself pinned to the compiled reference at 1e-12 in
test_oracle.py) and the reference's golden vectors.

The two sampling modes that make a step deterministic are checked: threshold_half
(pretrain.cpp:71-77) and injected uniforms (u < p, the reference's
sample_bernoulli with the Rng's draws supplied). A Bernoulli decision whose
probability sits within rounding of its threshold could flip between fp32 and
fp64, so at config-4 shapes the inputs are chosen with a margin: the hidden
biases are shifted per column so that no pre-activation is within 1e-4 of 0
(threshold), and injected uniforms are moved at least 1e-4 away from the fp64
probability. Every decision is then the reference's and the parameter deltas
are compared at fp32 tolerance.
"""
import numpy as np
import pytest

from conftest import rel
from oracle import parnn_oracle as O
from paper_1507_01239_b200 import parnn as P

pytestmark = pytest.mark.gpu

TOL = {P.Precision.fp32: 1e-5, P.Precision.tf32: 3e-3, P.Precision.bf16: 3e-2}


def f32(x):
    return np.asarray(x, np.float64).astype(np.float32).astype(np.float64)


def unpack(p, v, h):
    return p[:h * v].reshape(h, v), p[h * v:h * v + v], p[h * v + v:]


def blocks_rel(p_dev, p_ref, p0, v, h):
    """Relative L2 error of the parameter delta, per block (W, v_bias, h_bias)."""
    return [rel(a - c, b - c) for a, b, c in zip(unpack(p_dev, v, h), unpack(p_ref, v, h), unpack(p0, v, h))]


@pytest.mark.parametrize("prec", [P.Precision.fp32, P.Precision.tf32, P.Precision.bf16])
@pytest.mark.parametrize("kind,gauss", [("bern", False), ("gauss", True)])
def test_cd1_golden(ctx, golden, kind, gauss, prec):
    """The reference's own CD-1 golden vectors (v=6, h=4, 8 rows)."""
    v, h = 6, 4
    p0, batch = golden[f"rbm_{kind}_p0"], golden[f"rbm_{kind}_batch"]
    tol = TOL[prec]
    # the golden inputs are fp64; the device holds fp32, so compare with the
    # oracle on the fp32-rounded inputs at fp32 tolerance and with the golden
    # itself at the fp32 rounding of the inputs
    r = P.Rbm(ctx, v, h, gauss, batch=8, precision=prec)
    for mode in ("threshold", "uniforms"):
        r.set_params(p0)
        u = P.rng_uniform(99, batch.shape[0] * h)  # the reference's Rng(99) draws, injected
        r.cd1(batch, 0.1, sampling=mode, uniforms=u if mode == "uniforms" else None)
        got = r.get_params()
        rb = O.Rbm(*[x.copy() for x in unpack(f32(p0), v, h)], gauss)
        sampler = O.threshold_half if mode == "threshold" else (lambda p: (u.reshape(p.shape) < p).astype(float))
        pref = O.hidden_probs(rb, f32(batch))
        margin = np.abs(pref - (0.5 if mode == "threshold" else u.reshape(pref.shape))).min()
        if prec == P.Precision.bf16 and margin < 2e-2:
            continue  # a bf16 probability this close to its threshold may draw the other sample
        gold = golden[f"rbm_{kind}_thr_p" if mode == "threshold" else f"rbm_{kind}_rng_p"]
        assert rel(got - p0, gold - p0) < max(tol, 1e-6), (mode, rel(got - p0, gold - p0))
        pos, hs, rec, neg = O.cd1_gibbs(rb, f32(batch), sampler)
        o = O.cd1_apply(rb, f32(batch), pos, rec, neg, 0.1)
        ref = np.concatenate([o.W.ravel(), o.vb, o.hb])
        assert max(blocks_rel(got, ref, f32(p0), v, h)) < tol, (mode, blocks_rel(got, ref, f32(p0), v, h))
    r.set_params(p0)
    want = float(golden[f"rbm_{kind}_recerr"])
    assert abs(r.reconstruction_error(batch) - want) <= max(tol, 1e-6) * max(1.0, want)


def _cfg4_case(v, h, gauss, seed, b=128):
    rng = np.random.default_rng(seed)
    W = f32(rng.normal(0, 0.01, (h, v)))
    vb = f32(rng.normal(0, 0.01, v))
    hb = f32(rng.normal(0, 0.01, h))
    x = f32(rng.standard_normal((b, v)) if gauss else rng.random((b, v)))
    return W, vb, hb, x, rng


def _margin_hb(W, hb, x, margin=1e-4):
    """Shift each hidden bias so that no row's pre-activation is within
    `margin` of 0 (threshold_half decisions are then the same in fp32 and fp64)."""
    z = x @ W.T + hb
    out = hb.copy()
    cand = np.linspace(-0.02, 0.02, 401)
    for j in range(W.shape[0]):
        best = cand[np.argmax(np.abs(z[None, :, j] + cand[:, None]).min(axis=1))]
        out[j] = hb[j] + best
    out = f32(out)
    assert np.abs(x @ W.T + out).min() > margin
    return out


@pytest.mark.parametrize("prec", [P.Precision.fp32, P.Precision.tf32])
@pytest.mark.parametrize("v,h,gauss", [(440, 2048, True), (2048, 2048, False)])
def test_cd1_config4_shapes(ctx, v, h, gauss, prec):
    """Config-4 shapes (440->2048 Gaussian-Bernoulli, 2048->2048), batch 128,
    three consecutive CD-1 steps (threshold, uniforms, threshold) against the
    oracle run on the same fp32-rounded state."""
    W, vb, hb, x, rng = _cfg4_case(v, h, gauss, 7 + v)
    hb = _margin_hb(W, hb, x)
    p0 = np.concatenate([W.ravel(), vb, hb])
    r = P.Rbm(ctx, v, h, gauss, batch=128, precision=prec)
    r.set_params(p0)
    state = O.Rbm(W.copy(), vb.copy(), hb.copy(), gauss)
    lr = 0.1
    for step, mode in enumerate(("threshold", "uniforms", "threshold")):
        xs = x if step != 2 else f32(np.roll(x, 5, axis=0))
        if mode == "threshold" and step:
            # re-centre the device and oracle states on a margin-safe hb
            hbm = _margin_hb(state.W, f32(state.hb), xs)
            state = O.Rbm(f32(state.W), f32(state.vb), hbm, gauss)
            r.set_params(np.concatenate([state.W.ravel(), state.vb, state.hb]))
        before = np.concatenate([state.W.ravel(), state.vb, state.hb])
        if mode == "uniforms":
            p = O.hidden_probs(state, xs)
            u = rng.random(p.shape)
            near = np.abs(u - p) < 1e-4
            u[near] = np.where(p[near] > 0.5, p[near] - 2e-4, p[near] + 2e-4)
            sampler = lambda q, u=u: (u < q).astype(float)  # noqa: E731
            r.cd1(xs, lr, sampling="uniforms", uniforms=u.ravel())
        else:
            sampler = O.threshold_half
            r.cd1(xs, lr, sampling="threshold")
        pos, hs, rec, neg = O.cd1_gibbs(state, xs, sampler)
        state = O.cd1_apply(state, xs, pos, rec, neg, lr)
        ref = np.concatenate([state.W.ravel(), state.vb, state.hb])
        got = r.get_params()
        # per block: TOL relative to the update, plus 2 ulp of fp32 rounding of the
        # stored parameters (the reference keeps fp64; by step 2 the units saturate
        # and the update is ~1e-5 of W, below W's own fp32 ulp)
        for name, g, f, b0 in zip(("W", "v_bias", "h_bias"), unpack(got, v, h), unpack(ref, v, h),
                                  unpack(before, v, h)):
            err, bound = np.linalg.norm(g - f), TOL[prec] * np.linalg.norm(f - b0) + 2.0 ** -22 * np.linalg.norm(f)
            assert err <= bound, (step, mode, name, err, bound)
        # continue both from the device's fp32 state
        state = O.Rbm(*[a.copy() for a in unpack(got, v, h)], gauss)


@pytest.mark.parametrize("v,h,gauss", [(440, 2048, True), (2048, 2048, False)])
def test_hidden_probs_and_recerr_config4(ctx, v, h, gauss):
    W, vb, hb, x, _ = _cfg4_case(v, h, gauss, 3, b=300)  # 300 rows: two full chunks + a ragged one
    r = P.Rbm(ctx, v, h, gauss, batch=128, precision=P.Precision.fp32)
    r.set_params(np.concatenate([W.ravel(), vb, hb]))
    st = O.Rbm(W, vb, hb, gauss)
    assert np.abs(r.hidden_probs(x) - O.hidden_probs(st, x)).max() < 1e-6
    want = O.reconstruction_error(st, x)
    assert abs(r.reconstruction_error(x) - want) < 1e-5 * want


def test_cd1_philox_draws_are_bernoulli(ctx):
    """Counter-based Bernoulli draws: the fraction of 'on' samples of each
    hidden unit over a 1024-row batch matches its probability within 5 sigma,
    and two counters give different samples."""
    v, h, b = 64, 256, 1024
    hb = np.linspace(-3, 3, h)
    x = np.zeros((b, v))
    r = P.Rbm(ctx, v, h, False, batch=b, precision=P.Precision.fp32)
    # v = 0 rows: pos_j = sigmoid(hb_j); W = [I; 0] routes hidden sample j < v to
    # visible unit j, so recon_j = sigmoid(hs_j) is 0.5 or sigmoid(1)
    W = np.zeros((h, v))
    W[np.arange(v), np.arange(v)] = 1.0
    p0 = np.concatenate([W.ravel(), np.zeros(v), hb])
    outs = []
    for counter in (0, 1 << 40):
        r.set_params(p0)
        r.cd1(x, 1.0, sampling="philox", seed=11, counter=counter)
        outs.append(r.get_params())
    # vb += lr/b * sum(v - recon) = -mean(sigmoid(hs_j)) for j < v, so
    # mean(hs_j) follows from vb: sigmoid(1) * f + 0.5 * (1 - f) = -dvb
    s1 = 1 / (1 + np.exp(-1.0))
    for o in outs:
        dvb = o[h * v:h * v + v]
        f = (-dvb - 0.5) / (s1 - 0.5)
        p = 1 / (1 + np.exp(-hb[:v]))
        assert np.all(np.abs(f - p) < 5 * np.sqrt(p * (1 - p) / b) + 1e-6)
    assert not np.array_equal(outs[0], outs[1])


@pytest.mark.parametrize("prec", [P.Precision.bf16, P.Precision.fp32])
def test_greedy_pretrain_graphs_match_stream_launches(ctx, prec, monkeypatch):
    """The graph-launched epochs (32-step graphs with double-buffered batch rows
    gathered on a side stream and the bias update beside the weight update, plus
    single-step graphs for the remainder) give bit-identical parameters to the
    same CD-1 steps launched one kernel at a time (PARNN_CD1_GRAPH=0)."""
    rng = np.random.default_rng(4)
    x = rng.standard_normal((4500, 64))  # 35 steps of 128 per epoch: one 32-step graph + 3 single steps
    dims = [64, 96, 80, 10]
    opts = P.PretrainOptions(epochs=2)
    a = P.greedy_pretrain(dims, x, opts, seed=9, precision=prec, ctx=ctx).params
    monkeypatch.setenv("PARNN_CD1_GRAPH", "0")
    b = P.greedy_pretrain(dims, x, opts, seed=9, precision=prec, ctx=ctx).params
    assert np.array_equal(a, b)
    assert np.all(np.isfinite(a))


@pytest.mark.parametrize("prec", [P.Precision.fp32, P.Precision.bf16])
@pytest.mark.parametrize("v,h,b,gauss", [(300, 200, 37, False), (77, 130, 5, True), (129, 257, 128, False)])
def test_cd1_ragged_shapes(ctx, v, h, b, gauss, prec):
    """Ragged widths and batches (not multiples of 8 / 32 / 64, a partial row
    chunk, b < 8): one CD-1 step with margin-safe injected uniforms against the
    oracle (fp32 1e-5; bf16 with its own tolerance)."""
    rng = np.random.default_rng(v + h + b)
    W = f32(rng.normal(0, 0.05, (h, v)))
    vb = f32(rng.normal(0, 0.05, v))
    hb = f32(rng.normal(0, 0.05, h))
    x = f32(rng.standard_normal((b, v)) if gauss else rng.random((b, v)))
    p0 = np.concatenate([W.ravel(), vb, hb])
    st = O.Rbm(W.copy(), vb.copy(), hb.copy(), gauss)
    p = O.hidden_probs(st, x)
    u = rng.random(p.shape)
    margin = 1e-4 if prec == P.Precision.fp32 else 3e-2
    near = np.abs(u - p) < margin
    u[near] = np.clip(np.where(p[near] > 0.5, p[near] - 2 * margin, p[near] + 2 * margin), 0.0, 0.999999)
    r = P.Rbm(ctx, v, h, gauss, batch=128, precision=prec)
    r.set_params(p0)
    r.cd1(x, 0.1, sampling="uniforms", uniforms=u.ravel())
    pos, hs, rec, neg = O.cd1_gibbs(st, x, lambda q: (u < q).astype(float))
    ref = O.cd1_apply(st, x, pos, rec, neg, 0.1)
    got = r.get_params()
    refp = np.concatenate([ref.W.ravel(), ref.vb, ref.hb])
    errs = blocks_rel(got, refp, p0, v, h)
    assert max(errs) < TOL[prec], errs
