"""GPU tests of the model average (Averager, csrc/parallel.cu) on every branch
of its protocol (allreduce_average, parallel.cpp:40-59; train_loop's events,
parallel.cpp:195-214):

* the NCCL branches run on a 1-rank communicator on the single test GPU:
  one replica per process (in-place ncclAvg) and several (local midpoint tree
  -> ncclSum -> fused x 1/m + bf16 copy). Both must equal the local-tree path
  bitwise (a 1-rank sum is the identity);
* the per-layer buckets: averaging every step through the bucketed,
  event-gated path trains to exactly the same bits as an average issued only
  after every replica's step has finished;
* contribution-count errors carry the reference's message;
* averaging after every step with plain SGD equals one replica on the
  concatenated batch (gradient averaging).
"""
import numpy as np
import pytest

from conftest import rel
from oracle import parnn_oracle as O
from paper_1507_01239_b200 import parnn as P

pytestmark = pytest.mark.gpu

DIMS = [20, 33, 40, 7]


def _replicas(ctx, k, prec=P.Precision.bf16, seed0=100):
    x = np.random.default_rng(0).standard_normal((64, DIMS[0]))
    ds = P.DeviceDataset(ctx, P.Dataset(x, (np.arange(64) % DIMS[-1]).astype(np.int32), DIMS[-1]))
    reps, vecs = [], []
    for r in range(k):
        v = np.random.default_rng(seed0 + r).standard_normal(P.param_count(DIMS)).astype(np.float32).astype(np.float64)
        rp = P.Replica(ctx, DIMS, precision=prec, minibatch=16)
        rp.set_params(v)
        rp.bind(ds)
        reps.append(rp)
        vecs.append(v)
    return ds, reps, vecs


@pytest.fixture(scope="module")
def comm1(ctx):
    c = P.Comm(ctx, P.Comm.unique_id(), 1, 0)
    yield c
    c.close()


@pytest.mark.parametrize("k", [1, 2, 4, 8])
def test_nccl_branches_equal_local_tree(ctx, comm1, k):
    ds, reps, vecs = _replicas(ctx, k)
    _, reps_local, _ = _replicas(ctx, k)
    P.average(reps, comm=comm1, m_total=k)  # k == 1: ncclAvg; k > 1: tree -> ncclSum -> scale
    P.average(reps_local, m_total=k)        # local midpoint tree x 1/m
    out = [r.get_params() for r in reps]
    ref = reps_local[0].get_params()
    for o in out:
        assert np.array_equal(o, ref)
    if k > 1:
        t = O.tree_sum([v.astype(np.float32) for v in vecs], 0, k) * np.float32(1.0 / k)
        assert np.array_equal(ref.astype(np.float32), t.astype(np.float32))
    else:
        assert np.array_equal(out[0], vecs[0])
    # the bf16 operand copy was rebuilt with the averaged weights: the forward of
    # an averaged replica equals a fresh replica loaded with the average
    fresh = P.Replica(ctx, DIMS, precision=P.Precision.bf16, minibatch=16)
    fresh.set_params(ref)
    fresh.bind(ds)
    rows = np.arange(16)
    assert np.array_equal(reps[-1].forward(ds, rows), fresh.forward(ds, rows))


def test_contribution_count_errors(ctx, comm1):
    _, reps, _ = _replicas(ctx, 2)
    with pytest.raises(P.ParnnError, match="allreduce_average: got 2 contributions for m = 4"):
        P.average(reps, comm=comm1, m_total=4)
    with pytest.raises(P.ParnnError, match="allreduce_average: got 2 contributions for m = 3"):
        P.average(reps, m_total=3)


def test_train_with_one_rank_comm_matches_local(ctx, comm1, golden):
    """train_parallel through the NCCL branch (m = 4 workers hosted by one
    process of a 1-rank communicator) equals the purely local run bitwise."""
    dims = [int(d) for d in golden["dims"]]
    tr = P.Dataset(golden["data_tx"], golden["data_ty"], 10)
    cv = P.Dataset(golden["data_cx"], golden["data_cy"], 10)
    m0 = P.MlpModel(dims, P.Activation.sigmoid, golden["init_p0"])
    opts = P.TrainOptions(optimizer=P.OptimizerKind.sgd, lr_init=0.5, epochs=2, precision=P.Precision.fp32)
    plan = P.ParallelPlan(4, 2, 8, 17)
    a = P.train_parallel(plan, m0, tr, cv, opts, ctx=ctx)
    b = P.train_parallel(plan, m0, tr, cv, opts, ctx=ctx, comm=comm1)
    assert np.array_equal(a.model.params, b.model.params)
    assert [m.train_ce for m in a.metrics] == [m.train_ce for m in b.metrics]
    with pytest.raises(P.ParnnError, match="process 0 must host workers"):
        P.train_parallel(plan, m0, tr, cv, opts, ctx=ctx, comm=comm1, rank0=0, local_workers=2)


@pytest.mark.parametrize("opt", [P.OptimizerKind.sgd, P.OptimizerKind.ngsgd_lowrank])
def test_bucketed_average_equals_synchronous(ctx, opt):
    """Averaging every step through the per-layer buckets (each bucket starts
    when the step's update of that layer is recorded; the next step's forward
    of layer l waits on bucket l) gives the same bits as averaging only after
    all replicas' steps have finished (host synchronisation in between)."""
    dims = [40, 256, 192, 300]
    n = 1024
    x = np.random.default_rng(0).standard_normal((n, dims[0]))
    y = np.random.default_rng(1).integers(0, dims[-1], n).astype(np.int32)
    ds = P.DeviceDataset(ctx, P.Dataset(x, y, dims[-1]))
    m0 = P.init_random(dims, seed=3)
    k, steps, B = 4, 6, 64
    out = []
    for mode in ("bucketed", "sync"):
        reps = []
        for r in range(k):
            rp = P.Replica(ctx, dims, precision=P.Precision.bf16, optimizer=opt, minibatch=B, max_steps=steps)
            rp.set_params(m0.params)
            rp.bind(ds)
            rp.upload_epoch(np.random.default_rng(10 + r).integers(0, n, steps * B), np.full(steps, 0.1))
            reps.append(rp)
        if mode == "bucketed":
            P.run_steps(reps, steps, 1)  # average after every step, asynchronously
        else:
            for s in range(steps):
                for rp in reps:
                    rp.step(1)
                for rp in reps:
                    rp.sync()
                P.average(reps)
        out.append([rp.get_params() for rp in reps])
    for a, b in zip(*out):
        assert np.array_equal(a, b)


def test_time_average_reports_bytes(ctx):
    _, reps, _ = _replicas(ctx, 4)
    ms, nbytes = P.time_average(reps, iters=5)
    assert ms > 0
    assert nbytes >= 4 * reps[0].P  # fp32 bytes of the padded parameter layout


def test_averaging_every_step_equals_gradient_averaging(ctx):
    """SPEC.md:404 / SURVEY §8(c): with plain SGD and averaging after every step
    (K = 1), m replicas that start from the same parameters and each take one
    batch of B frames equal ONE replica stepping on the concatenated m*B frames
    (the average of m SGD updates is the SGD update of the batch-mean gradient).
    Config-1 layer widths, m = 4, B = 64, 5 steps, fp32 mode: the parameter
    deltas agree to fp32 rounding (the two sides sum in different orders)."""
    dims = [440, 512, 512, 1000]
    m, B, T = 4, 64, 5
    tr, _ = P.make_data(1000, 440, 4, 16.0, 7, 0.10, 2, True)
    ds = P.DeviceDataset(ctx, tr)
    p0 = P.init_random(dims, seed=1).params
    rng = np.random.default_rng(5)
    rows = rng.integers(0, tr.size(), (T, m, B))
    lrs = np.full(T, 0.5, np.float32)
    reps = []
    for r in range(m):
        rep = P.Replica(ctx, dims, precision=P.Precision.fp32, optimizer=P.OptimizerKind.sgd, minibatch=B,
                        max_steps=T)
        rep.set_params(p0)
        rep.bind(ds)
        rep.upload_epoch(rows[:, r, :].ravel(), lrs)
        reps.append(rep)
    P.run_steps(reps, T, 1)
    for rep in reps:
        rep.sync()
    avg = reps[0].get_params()
    for rep in reps[1:]:
        assert np.array_equal(rep.get_params(), avg)  # every replica holds the average
    one = P.Replica(ctx, dims, precision=P.Precision.fp32, optimizer=P.OptimizerKind.sgd, minibatch=m * B, max_steps=T)
    one.set_params(p0)
    one.bind(ds)
    one.upload_epoch(rows.reshape(T, m * B).ravel(), lrs)
    one.step(T)
    one.sync()
    big = one.get_params()
    assert rel(avg - p0, big - p0) < 1e-5, rel(avg - p0, big - p0)
    for rep in reps + [one]:
        rep.close()
