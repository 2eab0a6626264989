"""GPU parity tests: the CUDA path (through the C ABI) against the compiled
reference's golden fixtures and the numpy oracle, on identical seeds/data.

Tolerances (BASELINE.json north_star): per-layer parameter relative L2 within
1e-4 after one averaging period in fp32 mode (TF32 operands, fp32 accumulate,
fp32 NG solves); final frame CE within 1%. BF16 runs use looser, stated bounds.
Integer/index work (shards, batch order, events) is bit-exact.
"""
import numpy as np
import pytest

from conftest import rel
from oracle import parnn_oracle as O
from paper_1507_01239_b200 import parnn as P

pytestmark = pytest.mark.gpu

TF32, BF16, FP32 = P.Precision.tf32, P.Precision.bf16, P.Precision.fp32


def gdims(golden):
    return [int(d) for d in golden["dims"]]


def layer_rel(p, ref, dims):
    out, pos = [], 0
    for l in range(len(dims) - 1):
        n = dims[l] * dims[l + 1] + dims[l + 1]
        out.append(rel(p[pos:pos + n], ref[pos:pos + n]))
        pos += n
    return out


@pytest.mark.parametrize("prec,tol", [(FP32, 1e-5), (TF32, 2e-3), (BF16, 1.5e-2)])
def test_forward_ragged_shapes(ctx, prec, tol):
    dims = [37, 50, 29, 11]
    x = np.random.default_rng(0).standard_normal((90, 37))
    y = (np.arange(90) % 11).astype(np.int32)
    ds = P.DeviceDataset(ctx, P.Dataset(x, y, 11))
    m = P.init_random(dims, seed=5)
    r = P.Replica(ctx, dims, precision=prec, minibatch=45)
    r.set_params(m.params)
    r.bind(ds)
    rows = np.random.default_rng(1).permutation(90)[:45]
    z = r.forward(ds, rows)
    oz = O.forward(O.unflatten(m.params, dims), x[rows]).z[-1]
    assert rel(z, oz) < tol


@pytest.mark.parametrize("prec,theta_tol,dtheta_tol", [(FP32, 1e-4, 1e-3), (TF32, 3e-4, 5e-3), (BF16, 5e-4, 3e-2)])
def test_one_averaging_period_sgd(ctx, golden, prec, theta_tol, dtheta_tol):
    dims = gdims(golden)
    tr = P.Dataset(golden["data_tx"], golden["data_ty"], 10)
    ds = P.DeviceDataset(ctx, tr)
    r = P.Replica(ctx, dims, precision=prec, optimizer=P.OptimizerKind.sgd, minibatch=16, max_steps=4)
    r.set_params(golden["init_p0"])
    r.bind(ds)
    r.upload_epoch(golden["steps_rows"], golden["steps_lrs"])
    r.step(4)
    r.sync()
    p = r.get_params()
    ref = golden["steps_sgd_p"]
    assert max(layer_rel(p, ref, dims)) < theta_tol
    assert rel(p - golden["init_p0"], ref - golden["init_p0"]) < dtheta_tol
    assert np.abs(r.ce(4) - golden["steps_sgd_ce"]).max() < 5e-3 * np.abs(golden["steps_sgd_ce"]).max()


@pytest.mark.parametrize("prec,theta_tol,dtheta_tol,fac_tol", [(FP32, 1e-4, 2e-3, 1e-4), (TF32, 3e-4, 1e-2, 3e-3), (BF16, 1e-3, 5e-2, 2e-2)])
def test_one_averaging_period_ngsgd(ctx, golden, prec, theta_tol, dtheta_tol, fac_tol):
    dims = gdims(golden)
    ds = P.DeviceDataset(ctx, P.Dataset(golden["data_tx"], golden["data_ty"], 10))
    r = P.Replica(ctx, dims, precision=prec, optimizer=P.OptimizerKind.ngsgd, minibatch=16, max_steps=4)
    r.set_params(golden["init_p0"])
    r.bind(ds)
    r.upload_epoch(golden["steps_rows"], golden["steps_lrs"])
    r.step(4)
    r.sync()
    p = r.get_params()
    ref = golden["steps_ng_p"]
    assert max(layer_rel(p, ref, dims)) < theta_tol
    assert rel(p - golden["init_p0"], ref - golden["init_p0"]) < dtheta_tol
    for l, (ri, ro) in enumerate(r.get_ng_state()):
        assert rel(ri, golden[f"steps_ng_rin{l}"]) < fac_tol
        assert rel(ro, golden[f"steps_ng_rout{l}"]) < fac_tol


def test_ng_cold_start_is_sgd(ctx, golden):
    # SPEC: with a zero-history state the preconditioner reduces to identity after
    # rescaling -> one NG step with huge smoothing ~ one SGD step.
    dims = gdims(golden)
    ds = P.DeviceDataset(ctx, P.Dataset(golden["data_tx"], golden["data_ty"], 10))
    outs = []
    for opt, sm in ((P.OptimizerKind.sgd, 4.0), (P.OptimizerKind.ngsgd, 1e6)):
        r = P.Replica(ctx, dims, precision=FP32, optimizer=opt, minibatch=16, max_steps=1, ng_smoothing=sm)
        r.set_params(golden["init_p0"])
        r.bind(ds)
        r.upload_epoch(golden["steps_rows"][:16], [0.3])
        r.step(1)
        r.sync()
        outs.append(r.get_params() - golden["init_p0"])
    assert rel(outs[1], outs[0]) < 1e-3


def _train(ctx, golden, name, prec, **kw):
    dims = gdims(golden)
    tr = P.Dataset(golden["data_tx"], golden["data_ty"], 10)
    cv = P.Dataset(golden["data_cx"], golden["data_cy"], 10)
    m0 = P.MlpModel(dims, P.Activation.sigmoid, golden["init_p0"])
    ng = kw.pop("ngsgd")
    opts = P.TrainOptions(optimizer=P.OptimizerKind.ngsgd if ng else P.OptimizerKind.sgd,
                          lr_schedule=P.LrVariant.newbob if kw.pop("newbob", False) else P.LrVariant.exponential,
                          lr_init=kw.pop("lr_init", 0.32), epochs=kw.pop("epochs"), precision=prec)
    if kw.pop("serial", False):
        return P.serial_train(m0, tr, cv, opts, kw["minibatch"], 17, ctx=ctx)
    return P.train_parallel(P.ParallelPlan(kw["workers"], kw["avg_frequency"], kw["minibatch"], 17), m0, tr, cv, opts,
                            ctx=ctx)


RUNS = {
    "tp_sgd_m4": dict(workers=4, avg_frequency=2, minibatch=8, ngsgd=False, epochs=3, lr_init=0.5),
    "tp_ng_m2": dict(workers=2, avg_frequency=3, minibatch=8, ngsgd=True, epochs=2),
    "tp_sgd_newbob_m2": dict(workers=2, avg_frequency=4, minibatch=8, ngsgd=False, newbob=True, epochs=4, lr_init=0.5),
    "serial_sgd": dict(workers=1, avg_frequency=1, minibatch=8, ngsgd=False, epochs=2, lr_init=0.5, serial=True),
}


@pytest.mark.parametrize("name", sorted(RUNS))
def test_train_parallel_matches_reference(ctx, golden, name):
    res = _train(ctx, golden, name, FP32, **dict(RUNS[name]))
    ref = golden[f"{name}_met"]
    assert len(res.metrics) == ref.shape[0]
    for e, mt in enumerate(res.metrics):
        assert mt.epoch == ref[e, 0] and mt.workers == ref[e, 5] and mt.avg_events == ref[e, 6]
        assert abs(mt.lr - ref[e, 1]) <= 1e-15 * max(1.0, ref[e, 1])
        assert abs(mt.train_ce - ref[e, 2]) <= 0.01 * ref[e, 2]  # final-CE gate: within 1%
        # CV accuracy over 20 frames: at most one frame's argmax may flip between fp32 and fp64
        assert abs(mt.cv_accuracy - ref[e, 3]) <= 1.0 / golden["data_cx"].shape[0] + 1e-12
    assert rel(res.model.params, golden[f"{name}_p"]) < 2e-3


def test_serial_equals_parallel_m1_and_is_deterministic(ctx, golden):
    a = _train(ctx, golden, "s", FP32, workers=1, avg_frequency=1, minibatch=8, ngsgd=True, epochs=1, serial=True)
    b = _train(ctx, golden, "p", FP32, workers=1, avg_frequency=1, minibatch=8, ngsgd=True, epochs=1)
    c = _train(ctx, golden, "p", FP32, workers=1, avg_frequency=1, minibatch=8, ngsgd=True, epochs=1)
    assert np.array_equal(a.model.params, b.model.params)
    assert np.array_equal(b.model.params, c.model.params)


@pytest.mark.parametrize("m", [2, 3, 4, 5, 8, 16, 32])
def test_device_average_matches_tree(ctx, m):
    dims = [20, 33, 7]
    x = np.random.default_rng(0).standard_normal((40, 20))
    ds = P.DeviceDataset(ctx, P.Dataset(x, (np.arange(40) % 7).astype(np.int32), 7))
    reps, vecs = [], []
    for r in range(m):
        v = np.random.default_rng(100 + r).standard_normal(P.param_count(dims)).astype(np.float32).astype(np.float64)
        rp = P.Replica(ctx, dims, precision=BF16, minibatch=8)
        rp.set_params(v)
        rp.bind(ds)
        reps.append(rp)
        vecs.append(v)
    P.average(reps)
    out = [rp.get_params() for rp in reps]
    ref = O.allreduce_average(vecs, m)
    for o in out:
        assert np.array_equal(o, out[0])  # every worker sees the identical vector
    assert np.abs(out[0] - ref).max() < 1e-6 * max(1.0, np.abs(ref).max())
    if m in (2, 4, 8, 16, 32):  # power of two: fp32 tree sum of fp32 inputs, exact scale
        t = O.tree_sum([v.astype(np.float32) for v in vecs], 0, m) * np.float32(1.0 / m)
        assert np.array_equal(out[0].astype(np.float32), t.astype(np.float32))


def test_ng_cholesky_failure_matches_reference(ctx, golden, reflib):
    """A NaN frame under NG-SGD: the reference fails in ng_precondition's
    Cholesky (matrix.cpp:110-113) before sgd_step's check, and so does the
    device factorization -- the same message, pivot value and index."""
    dims = gdims(golden)
    x = golden["data_tx"].copy()
    x[3, 2] = np.nan
    tr = P.Dataset(x, golden["data_ty"], 10)
    cv = P.Dataset(golden["data_cx"], golden["data_cy"], 10)
    m0 = P.MlpModel(dims, P.Activation.sigmoid, golden["init_p0"])
    with pytest.raises(RuntimeError) as ref_err:
        reflib.train_parallel(dims, golden["init_p0"], x, golden["data_ty"], golden["data_cx"], golden["data_cy"],
                              workers=1, avg_frequency=1, minibatch=16, base_seed=0, ngsgd=True, epochs=1)
    opts = P.TrainOptions(optimizer=P.OptimizerKind.ngsgd, epochs=1, precision=FP32)
    with pytest.raises(P.ParnnError) as ours:
        P.train_parallel(P.ParallelPlan(1, 1, 16, 0), m0, tr, cv, opts, ctx=ctx)
    assert str(ours.value) == str(ref_err.value)
    assert "cholesky_solve: non-positive-definite pivot -nan at index 0" in str(ours.value)


def test_nonfinite_gradient_names_layer(ctx, golden):
    dims = gdims(golden)
    x = golden["data_tx"].copy()
    x[3, 2] = np.nan
    ds = P.DeviceDataset(ctx, P.Dataset(x, golden["data_ty"], 10))
    r = P.Replica(ctx, dims, precision=TF32, minibatch=16, max_steps=1)
    r.set_params(golden["init_p0"])
    r.bind(ds)
    rows = np.arange(16)
    r.upload_epoch(rows, [0.1])
    r.step(1)
    with pytest.raises(P.ParnnError, match=r"sgd_step: non-finite weight gradient in layer 0"):
        r.sync()


def test_errors_cross_the_abi(ctx, golden):
    dims = gdims(golden)
    with pytest.raises(P.ParnnError, match="ng_init: decay must be in"):
        P.Replica(ctx, dims, ng_decay=1.5)
    tr = P.Dataset(golden["data_tx"], golden["data_ty"], 10)
    m0 = P.MlpModel(dims, P.Activation.sigmoid, golden["init_p0"])
    with pytest.raises(P.ParnnError, match="train_parallel: empty CV set"):
        P.train_parallel(P.ParallelPlan(2, 2, 8, 0), m0, tr, P.Dataset(np.zeros((0, 12)), np.zeros(0, np.int32), 10),
                         P.TrainOptions(epochs=1), ctx=ctx)
    cv = P.Dataset(golden["data_cx"], golden["data_cy"], 10)
    with pytest.raises(P.ParnnError, match="worker rank 0 failed: minibatches: batch size 500 exceeds dataset size 90"):
        P.train_parallel(P.ParallelPlan(2, 2, 500, 0), m0, tr, cv, P.TrainOptions(epochs=1), ctx=ctx)


@pytest.mark.parametrize("kind,gauss", [("bern", False), ("gauss", True)])
def test_rbm_cd1_parity_modes(ctx, golden, kind, gauss):
    v, h = 6, 4
    p0, batch = golden[f"rbm_{kind}_p0"], golden[f"rbm_{kind}_batch"]
    r = P.Rbm(ctx, v, h, gauss, batch=8, precision=TF32)
    r.set_params(p0)
    r.cd1(batch, 0.1, sampling="threshold")
    assert rel(r.get_params() - p0, golden[f"rbm_{kind}_thr_p"] - p0) < 1e-2
    r.set_params(p0)
    u = P.rng_uniform(99, batch.shape[0] * h)  # the reference's Rng(99) draws, injected
    r.cd1(batch, 0.1, sampling="uniforms", uniforms=u)
    assert rel(r.get_params() - p0, golden[f"rbm_{kind}_rng_p"] - p0) < 1e-2
    r.set_params(p0)
    assert abs(r.reconstruction_error(batch) - float(golden[f"rbm_{kind}_recerr"])) < 1e-3 * max(
        1.0, float(golden[f"rbm_{kind}_recerr"]))


def test_rbm_philox_statistics(ctx):
    # counter-based sampling: reconstruction error falls on a 2-cluster set
    rng = np.random.default_rng(0)
    x = (rng.random((512, 16)) < np.where(np.arange(512)[:, None] % 2 == 0, 0.9, 0.1)).astype(np.float64)
    r = P.Rbm(ctx, 16, 8, False, batch=64, precision=TF32)
    r.set_params(np.concatenate([rng.normal(0, 0.01, 128), np.zeros(24)]))
    e0 = r.reconstruction_error(x)
    for ep in range(20):
        for b in range(8):
            r.cd1(x[b * 64:(b + 1) * 64], 0.1, sampling="philox", seed=5, counter=(ep * 8 + b) * 64 * 8)
    assert r.reconstruction_error(x) < 0.8 * e0


def test_greedy_pretrain_rng_stream(ctx, golden):
    # Host Rng consumption matches the reference exactly (GF(2) jump over the
    # Bernoulli draws), so the output layer's Glorot init is bit-identical.
    dims = [int(d) for d in golden["pre_dims"]]
    m = P.greedy_pretrain(dims, golden["data_tx"][:64], P.PretrainOptions(epochs=2, batch_size=8), seed=41, ctx=ctx)
    ref = golden["pre_p"]
    n_out = dims[-2] * dims[-1] + dims[-1]
    assert np.array_equal(m.params[-n_out:], ref[-n_out:])
    assert np.all(np.isfinite(m.params))
    # first RBM layer stays close to the reference (only the Bernoulli draws differ)
    n0 = dims[0] * dims[1]
    assert rel(m.params[:n0], ref[:n0]) < 0.5


@pytest.mark.parametrize("prec", [BF16, TF32, FP32])
@pytest.mark.parametrize("opt", [P.OptimizerKind.sgd, P.OptimizerKind.ngsgd])
def test_config2_shape_step(ctx, prec, opt):
    dims = [440] + [2048] * 6 + [8806]
    n = 4096
    x = np.random.default_rng(0).standard_normal((n, 440))
    y = np.random.default_rng(1).integers(0, 8806, n).astype(np.int32)
    ds = P.DeviceDataset(ctx, P.Dataset(x, y, 8806))
    r = P.Replica(ctx, dims, precision=prec, optimizer=opt, minibatch=1024, max_steps=2)
    r.set_params(P.init_random(dims, seed=1).params)
    r.bind(ds)
    r.upload_epoch(np.random.default_rng(2).integers(0, n, 2048), [0.01, 0.01])
    r.step(2)
    r.sync()
    ce = r.ce(2)
    assert np.all(np.isfinite(ce)) and abs(ce[0] - np.log(8806)) < 0.2
    assert r.kernels_per_step() > 15


def test_reference_adapter_dropin():
    # The reference's own C++ types + train_parallel (from its unmodified
    # sources) next to the C-ABI adapter (integration/), same inputs.
    import json
    import os
    import subprocess
    exe = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "integration", "_build",
                       "adapter_demo")
    if not os.path.exists(exe):
        pytest.skip("integration/_build/adapter_demo not built (needs the reference headers at build time)")
    out = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stderr
    res, low, pre, err = [json.loads(l) for l in out.stdout.strip().splitlines()]
    assert res["epochs"][0] == res["epochs"][1] and res["avg_events"][0] == res["avg_events"][1]
    assert abs(res["ce_ref"] - res["ce_b200"]) <= 0.01 * res["ce_ref"]
    assert res["theta_rel_l2"] < 2e-3
    # the low-rank NG-SGD selected through the same adapter trains as well as the reference's NG
    assert low["lowrank_epochs"] == res["epochs"][0]
    assert np.isfinite(low["ce_lowrank"]) and low["ce_lowrank"] <= 1.05 * low["ce_ref"]
    assert "train_parallel: avg_frequency must be >= 1" in err["error"]
    # greedy_pretrain drop-in: the caller's Rng (incl. a cached gaussian spare) crosses the ABI
    # and comes back in the reference's state; the output layer is bit-identical
    assert pre["pretrain_output_layer_equal"] and pre["pretrain_rng_state_equal"] and pre["activation_equal"]
    assert pre["pretrain_layer0_rel_l2"] < 0.5  # CD-1 Bernoulli draws differ (counter-based RNG)


_PATH_SCRIPT = r"""
import sys, numpy as np
sys.path.insert(0, sys.argv[1])
from paper_1507_01239_b200 import parnn as P
ctx = P.Context(0)
dims = [440, 2048, 2048, 1101]
x = np.random.default_rng(0).standard_normal((4096, 440))
y = np.random.default_rng(1).integers(0, 1101, 4096).astype(np.int32)
ds = P.DeviceDataset(ctx, P.Dataset(x, y, 1101))
r = P.Replica(ctx, dims, precision=P.Precision.bf16, optimizer=P.OptimizerKind.sgd, minibatch=1024, max_steps=3)
r.set_params(P.init_random(dims, seed=1).params)
r.bind(ds)
r.upload_epoch(np.random.default_rng(2).integers(0, 4096, 3 * 1024), [0.05] * 3)
r.step(3)
r.sync()
np.save(sys.argv[2], r.get_params())
"""


@pytest.mark.parametrize("var,alt", [("PARNN_GEMM_PAIRS", "1"), ("PARNN_GEMM_SK2", "0")])
def test_gemm_cluster_paths_match(tmp_path, var, alt):
    """The GEMM's cluster paths train to the same parameters as the plain 1-SM
    tiles (bf16 mode: the products are identical, only the fp32 accumulation
    order differs): the opt-in 2-SM cta_group::2 pairs (PARNN_GEMM_PAIRS=1) and
    the default split-K pairs with the DSMEM partial-tile exchange, which the
    1024 x 2048 hidden GEMMs take (PARNN_GEMM_SK2=0 turns them off). The
    switches are read once per process, so each run is a subprocess."""
    import os
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = {}
    for v in ("default", alt):
        env = dict(os.environ)
        env.pop(var, None)
        if v != "default":
            env[var] = v
        f = tmp_path / f"p_{v}.npy"
        subprocess.run([sys.executable, "-c", _PATH_SCRIPT, root, str(f)], env=env, check=True, timeout=300)
        out[v] = np.load(f)
    d = np.linalg.norm(out[alt] - out["default"]) / np.linalg.norm(out["default"])
    assert d < 1e-4, d


_GROUP_SCRIPT = r"""
import sys, numpy as np
sys.path.insert(0, sys.argv[1])
from paper_1507_01239_b200 import parnn as P
ctx = P.Context(0)
dims = [440, 2048, 2048, 1101]
x = np.random.default_rng(0).standard_normal((4096, 440))
y = np.random.default_rng(1).integers(0, 1101, 4096).astype(np.int32)
ds = P.DeviceDataset(ctx, P.Dataset(x, y, 1101))
out = []
for opt in (P.OptimizerKind.sgd, P.OptimizerKind.ngsgd_lowrank):
    r = P.Replica(ctx, dims, precision=P.Precision.bf16, optimizer=opt, minibatch=1024, max_steps=6)
    r.set_params(P.init_random(dims, seed=1).params)
    r.bind(ds)
    r.upload_epoch(np.random.default_rng(2).integers(0, 4096, 6 * 1024), [0.05] * 6)
    r.step(6)
    r.sync()
    out.append(r.get_params())
np.save(sys.argv[2], np.concatenate(out))
"""


def test_grouped_dw_matches_per_layer(tmp_path):
    """Every layer's dW + SGD update in one grouped persistent launch (the
    default in bf16) gives exactly the parameters of one launch per layer
    (PARNN_NO_DW_GROUP=1): the tiles, their k-order and epilogues are the same;
    SGD and low-rank NG-SGD (bias column in the dW GEMM), 6 steps."""
    import os
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = {}
    for v in ("group", "per_layer"):
        env = dict(os.environ)
        env.pop("PARNN_NO_DW_GROUP", None)
        if v == "per_layer":
            env["PARNN_NO_DW_GROUP"] = "1"
        f = tmp_path / f"p_{v}.npy"
        subprocess.run([sys.executable, "-c", _GROUP_SCRIPT, root, str(f)], env=env, check=True, timeout=300)
        out[v] = np.load(f)
    assert np.array_equal(out["group"], out["per_layer"])
