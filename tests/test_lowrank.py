"""Low-rank online NG-SGD: oracle properties, host
basis parity, and GPU parity against oracle/ng_lowrank.py.

The reference has no low-rank NG, so parity is anchored on the oracle's
restatement of Povey et al. 2014 (parity unpinned) plus a
statistical gate against the reference's kron-full NG-SGD.
"""
import numpy as np
import pytest

from conftest import rel
from oracle import ng_lowrank as LR
from oracle import parnn_oracle as O


def _data(classes=12, dim=40, per_class=40, seed=1):
    x, y = O.generate_synthetic(classes, dim, per_class, 4.0, seed)
    mean, sd = O.feature_stats(x)
    return O.standardize(x, mean, sd), y


def _batches(n, B, steps, seed=0):
    perm = np.random.default_rng(seed).permutation(n)
    return [perm[(i * B + np.arange(B)) % n] for i in range(steps)]


# ------------------------------------------------------------------ CPU
def test_basis_capi_matches_oracle():
    from paper_1507_01239_b200 import parnn as P
    for dim, rank, l, side in [(13, 4, 0, 0), (41, 8, 2, 1), (97, 20, 5, 0)]:
        seed = LR.basis_seed(l, side)
        assert P.lowrank_seed(l, side) == seed
        b = P.lowrank_basis(dim, rank, seed)
        ob = LR.lowrank_basis(dim, rank, seed)
        assert rel(b, ob) < 1e-13
        assert np.abs(b @ b.T - np.eye(rank)).max() < 1e-13


def test_basis_rejects_bad_rank():
    from paper_1507_01239_b200 import parnn as P
    from paper_1507_01239_b200._lib import ParnnError
    with pytest.raises(ParnnError, match="lowrank_basis: need 0 < rank < dim"):
        P.lowrank_basis(8, 8, 1)


def test_oracle_preconditioner_invariants():
    rng = np.random.default_rng(3)
    cfg = LR.LowRankConfig(rank_in=5, rank_out=5, update_period=1)
    st = LR.side_init(30, 5, 7, cfg.alpha)
    # a correlated source: a few strong directions plus isotropic noise
    mix = rng.standard_normal((6, 30)) * 3.0
    for t in range(8):
        x = rng.standard_normal((64, 6)) @ mix + rng.standard_normal((64, 30))
        xh, g = LR.side_step(st, x, cfg)
        assert np.isclose(np.linalg.norm(g * xh), np.linalg.norm(x), rtol=1e-12)  # gamma keeps ||X||_F
        # W W^T = E (orthonormal R), eigenvalues sorted, floors respected
        assert np.abs(st.W @ st.W.T - np.diag(st.e)).max() < 1e-10
        assert np.all(np.diff(st.d) <= 1e-12) and st.d.min() >= LR.EPS and st.rho >= LR.EPS
    # the learned subspace captures the strong directions: their energy is damped most
    q, _ = np.linalg.qr(mix.T)
    rn = st.W / np.sqrt(st.e)[:, None]  # R_t: orthonormal rows
    captured = np.trace(q.T @ rn.T @ rn @ q) / st.rank
    assert captured > 0.95


def test_oracle_zero_state_is_identity():
    st = LR.side_init(20, 4, 1, 4.0)
    st.W[:] = 0.0
    x = np.random.default_rng(0).standard_normal((16, 20))
    h, xh, g, trxx = LR.precondition(st, x)
    assert np.array_equal(xh, x) and g == 1.0 and np.allclose(trxx, (x * x).sum())


def test_oracle_lowrank_tracks_kron_full():
    """Statistical gate of A17: low-rank NG-SGD reaches the reference kron-full
    NG-SGD's training CE on the same data and minibatch order."""
    x, y = _data()
    dims = [40, 48, 36, 12]
    m0 = O.init_random(dims, 0, O.Rng(3))
    batches = _batches(x.shape[0], 32, 60)
    lrs = [0.32] * len(batches)
    mk, ng = m0.copy(), O.ng_init(m0)
    ce_k = []
    for rows in batches:
        tr = O.forward(mk, x[rows])
        ce_k.append(O.cross_entropy(tr, y[rows]))
        gW, gb, dzs = O.backward(mk, tr, y[rows], want_dz=True)
        O.ng_update_state(ng, tr, dzs)
        gW, gb = O.ng_precondition(ng, gW, gb)
        O.sgd_step(mk, gW, gb, 0.32)
    ml = m0.copy()
    st = LR.lowrank_init(ml, LR.LowRankConfig(rank_in=8, rank_out=8, update_period=2))
    ce_l = LR.lowrank_train_steps(ml, st, x, y, batches, lrs)
    k, l = np.mean(ce_k[-10:]), np.mean(ce_l[-10:])
    assert l < ce_l[0] - 0.3  # it learns
    assert l < 1.05 * k  # at least as good as kron-full, to 5%


# ------------------------------------------------------------------ GPU
def _gpu_run(ctx, prec, x, y, dims, B, batches, lrs, cfg, steps_per_call=None):
    from paper_1507_01239_b200 import parnn as P
    ds = P.DeviceDataset(ctx, P.Dataset(x, y.astype(np.int32), dims[-1]))
    m = P.init_random(dims, seed=3)
    r = P.Replica(ctx, dims, precision=prec, optimizer=P.OptimizerKind.ngsgd_lowrank, minibatch=B,
                  max_steps=len(batches), ng_smoothing=cfg.alpha)
    r.set_lowrank(cfg.rank_in, cfg.rank_out, cfg.update_period, cfg.init_iters, cfg.num_samples_history,
                  cfg.update_lag)
    r.set_params(m.params)
    r.bind(ds)
    r.upload_epoch(np.concatenate(batches), lrs)
    if steps_per_call:
        for _ in range(len(batches) // steps_per_call):
            r.step(steps_per_call)
    else:
        r.step(len(batches))
    r.sync()
    return r, m.params, r.get_params(), r.ce(len(batches))


def _oracle_run(p0, dims, x, y, batches, lrs, cfg):
    m = O.unflatten(p0, dims)
    st = LR.lowrank_init(m, cfg)
    ces = LR.lowrank_train_steps(m, st, x, y, batches, lrs)
    return m, st, ces


@pytest.mark.gpu
@pytest.mark.parametrize("lag,period", [(1, 2), (2, 2), (3, 3), (4, 4)])
@pytest.mark.parametrize("prec,dtol", [("fp32", 2e-3), ("tf32", 3e-2), ("bf16", 8e-2)])
def test_lowrank_step_parity(ctx, prec, dtol, lag, period):
    from paper_1507_01239_b200 import parnn as P
    x, y = _data()
    dims = [40, 48, 36, 12]
    B = 32
    batches = _batches(x.shape[0], B, 6)
    lrs = np.array([0.32, 0.3, 0.28, 0.26, 0.24, 0.22], np.float32)
    cfg = LR.LowRankConfig(rank_in=6, rank_out=8, update_period=period, init_iters=3, update_lag=lag)
    r, p0, p, ce = _gpu_run(ctx, P.Precision[prec], x, y, dims, B, batches, lrs, cfg)
    mo, st, ce_o = _oracle_run(p0, dims, x, y, batches, lrs.astype(np.float64), cfg)
    po = O.flatten(mo)
    assert rel(p - p0, po - p0) < dtol
    assert np.abs(ce - np.array(ce_o)).max() < 1e-3 * max(ce_o)
    if prec == "fp32":
        assert rel(p, po) < 1e-4  # north-star fp32 gate (per-model relative L2)
        for l in range(len(dims) - 1):
            for side, so in ((0, st.sides_in[l]), (1, st.sides_out[l])):
                w, d, rho = r.lowrank_state(l, side)
                assert w.shape == so.W.shape
                assert rel(w.T @ w, so.W.T @ so.W) < 2e-3  # sign/rotation-invariant
                # rho = (tr T - sum c)/(D - R) amplifies fp32 differences ~5x on sides whose
                # d sit at the floors (the last layer's input side here): 1e-2
                assert rel(d, so.d) < 2e-3 and abs(rho - so.rho) / so.rho < 1e-2


@pytest.mark.gpu
def test_lowrank_graph_variants_deterministic(ctx):
    """Step-by-step launches (graph variant chosen per step) equal one
    multi-step call bit for bit, and reruns are bitwise identical."""
    from paper_1507_01239_b200 import parnn as P
    x, y = _data()
    dims = [40, 48, 36, 12]
    batches = _batches(x.shape[0], 32, 9)
    lrs = np.full(9, 0.3, np.float32)
    cfg = LR.LowRankConfig(rank_in=6, rank_out=8, update_period=3, init_iters=2, update_lag=2)
    _, _, p1, c1 = _gpu_run(ctx, P.Precision.bf16, x, y, dims, 32, batches, lrs, cfg)
    _, _, p2, c2 = _gpu_run(ctx, P.Precision.bf16, x, y, dims, 32, batches, lrs, cfg, steps_per_call=1)
    _, _, p3, _ = _gpu_run(ctx, P.Precision.bf16, x, y, dims, 32, batches, lrs, cfg, steps_per_call=3)
    assert np.array_equal(p1, p2) and np.array_equal(p1, p3) and np.array_equal(c1, c2)


@pytest.mark.gpu
def test_lowrank_train_parallel_vs_kron_reference(ctx, golden):
    """train_parallel with the low-rank optimizer against the reference's
    kron-full NG-SGD (golden tp_ng_m2 run): same epochs/events, final CE no
    worse than 5% above it (statistical gate; different preconditioners)."""
    from paper_1507_01239_b200 import parnn as P
    dims = [int(d) for d in golden["dims"]]
    tr = P.Dataset(golden["data_tx"], golden["data_ty"], 10)
    cv = P.Dataset(golden["data_cx"], golden["data_cy"], 10)
    m0 = P.MlpModel(dims, P.Activation.sigmoid, golden["init_p0"])
    plan = P.ParallelPlan(2, 3, 8, 17)  # the golden tp_ng_m2 plan (tests/golden/make_golden.py)
    opts = P.TrainOptions(optimizer=P.OptimizerKind.ngsgd_lowrank, epochs=2, lr_init=0.32,
                          precision=P.Precision.fp32, ng_rank_in=4, ng_rank_out=4, ng_update_period=2)
    res = P.train_parallel(plan, m0, tr, cv, opts, ctx=ctx)
    ref_ce = golden["tp_ng_m2_met"][:, 2]
    ce = np.array([m.train_ce for m in res.metrics])
    assert len(ce) == len(ref_ce)
    assert [m.avg_events for m in res.metrics] == [int(v) for v in golden["tp_ng_m2_met"][:, 6]]
    assert ce[-1] < 1.05 * ref_ce[-1]


@pytest.mark.gpu
@pytest.mark.parametrize("prec", ["bf16", "fp32"])
def test_lowrank_config2_shape_steps(ctx, prec):
    """Config-2 shapes (440-2048x6-8806, B=1024): default ranks, the init
    step, update and plain steps run and stay finite; CE decreases on a
    repeated batch."""
    from paper_1507_01239_b200 import parnn as P
    dims = [440] + [2048] * 6 + [8806]
    rng = np.random.default_rng(0)
    n = 2048
    x = rng.standard_normal((n, 440))
    y = (np.arange(n) % 8806).astype(np.int32)
    ds = P.DeviceDataset(ctx, P.Dataset(x, y, 8806))
    r = P.Replica(ctx, dims, precision=P.Precision[prec], optimizer=P.OptimizerKind.ngsgd_lowrank, minibatch=1024,
                  max_steps=6)
    r.set_params(P.init_random(dims, seed=1).params)
    r.bind(ds)
    rows = np.concatenate([np.arange(1024)] * 6)
    r.upload_epoch(rows, np.full(6, 0.32, np.float32))
    r.step(6)
    r.sync()
    ce = r.ce(6)
    assert np.all(np.isfinite(ce)) and ce[-1] < ce[0]
    assert np.all(np.isfinite(r.get_params()))
    assert r.kernels_per_step() > 0


@pytest.mark.gpu
@pytest.mark.parametrize("kind", ["isotropic", "mean_dominated", "decaying"])
@pytest.mark.parametrize("R", [20, 80])
def test_lowrank_eig_kernel_matches_oracle(kind, R):
    """The device eigensolver of the subspace update (one-sided Jacobi) against
    numpy eigh on the same Gram: new d, rho exactly (1e-6) and the updated
    basis W' = M [J; W] up to row signs (W'^T W')."""
    import ctypes as C
    from paper_1507_01239_b200 import parnn as P
    from paper_1507_01239_b200._lib import check, lib, ptr
    rng = np.random.default_rng(R)
    D, N = 2048, 1024
    if kind == "isotropic":
        x = rng.standard_normal((N, D)) * 1e-2
    elif kind == "mean_dominated":
        x = 1 / (1 + np.exp(-(rng.standard_normal((N, D)) * 1.5 + rng.standard_normal(D))))
    else:
        x = rng.standard_normal((N, D)) * (1.0 / (1 + np.arange(D)) ** 0.7)
    st = LR.side_init(D, R, 5, 4.0)
    cfg = LR.LowRankConfig(rank_in=R, update_period=1)
    eta = LR.eta_of(N, cfg)
    for _ in range(2):  # move away from the cold start
        h, _, _, trxx = LR.precondition(st, x)
        LR.update(st, x, h, trxx, eta, 4.0)
    h, _, _, trxx = LR.precondition(st, x)
    j = h.T @ x
    Y = np.concatenate([j, st.W], axis=0).astype(np.float32)
    gram = (Y.astype(np.float64) @ Y.astype(np.float64).T).astype(np.float32)
    a = eta / N
    d1, rho1, e1, m = LR.eig_update(st.d, st.e, st.rho, gram[:R, :R].astype(np.float64),
                                    gram[R:, :R].astype(np.float64), gram[R:, R:].astype(np.float64), trxx, D, eta,
                                    a, 4.0)
    sin = np.zeros(2 * R + 12)
    sin[:R], sin[R:2 * R], sin[2 * R], sin[2 * R + 1] = st.d, st.e, st.rho, trxx
    sout = np.zeros(2 * R + 12)
    mg = np.zeros((R, 2 * R), np.float32)
    sw = C.c_int()
    g32 = np.ascontiguousarray(gram, np.float32)
    check(lib().parnn_debug_lowrank_eig(R, D, eta, a, 4.0, ptr(sin), ptr(g32), ptr(sout), ptr(mg), C.byref(sw)))
    assert 0 < sw.value < 40
    assert rel(sout[:R], d1) < 1e-5 and abs(sout[2 * R] - rho1) / rho1 < 1e-5
    w_ref = m @ Y.astype(np.float64)
    w_gpu = mg.astype(np.float64) @ Y.astype(np.float64)
    assert rel(w_gpu.T @ w_gpu, w_ref.T @ w_ref) < 1e-4
