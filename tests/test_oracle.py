"""Pins the numpy restatement (oracle/parnn_oracle.py) against the golden
fixtures produced by the compiled reference (tests/golden/make_golden.py) and
against the known-answer examples of /root/reference/SPEC.md."""
import math

import numpy as np
import pytest

from conftest import rel
from oracle import parnn_oracle as O


def test_rng_streams_bit_exact(golden):
    r = O.Rng(7)
    assert np.array_equal(np.array([r.next_u64() for _ in range(64)], np.uint64), golden["rng_u64_s7"])
    r = O.Rng(11)
    assert np.array_equal(np.array([r.uniform() for _ in range(64)]), golden["rng_uniform_s11"])
    r = O.Rng(3)
    assert np.array_equal(np.array([r.gaussian(0.0, 1.0) for _ in range(101)]), golden["rng_gauss_s3"])
    r = O.Rng(5)
    assert np.array_equal(np.array([r.uniform_index(10) for _ in range(100)], np.uint64), golden["rng_index_s5_b10"])


def test_gaussian_zero_stddev_consumes_nothing():
    a, b = O.Rng(1), O.Rng(1)
    assert a.gaussian(2.5, 0.0) == 2.5
    assert a.next_u64() == b.next_u64()


def test_shuffles_partitions_minibatches_bit_exact(golden):
    assert np.array_equal(O.shuffled_indices(1000, 5), golden["shuffle_1000_s5"])
    assert np.array_equal(np.stack(O.partition_rows(10, 3, 9)), golden["partition_10_3_s9"])
    assert np.array_equal(np.stack(O.partition_rows(1000, 7, 11)), golden["partition_1000_7_s11"])
    assert np.array_equal(np.stack(O.minibatch_rows(10, 3, 11)), golden["minibatch_10_3_s11"])
    assert np.array_equal(np.stack(O.minibatch_rows(500, 32, 13)), golden["minibatch_500_32_s13"])


def test_spec_partition_and_minibatch_examples():
    # SPEC.md:382 (N=10, m=3 -> 3 shards of 3, one example dropped), :477 (N=10, B=3)
    sh = O.partition_rows(10, 3, 0)
    assert [len(s) for s in sh] == [3, 3, 3]
    assert len(set(np.concatenate(sh).tolist())) == 9
    assert np.array_equal(np.concatenate(sh), O.shuffled_indices(10, 0)[:9])
    assert len(O.minibatch_rows(10, 3, 0)) == 3
    with pytest.raises(ValueError, match="exceeds dataset size"):
        O.partition_rows(3, 4, 0)


def test_synthetic_data_split_standardize(golden):
    x, y = O.generate_synthetic(10, 12, 20, 4.0, 1)
    (tx, ty), (cx, cy) = O.split_cv(x, y, 0.1, 2)
    mu, sd = O.feature_stats(tx)
    tx, cx = O.standardize(tx, mu, sd), O.standardize(cx, mu, sd)
    assert np.array_equal(ty, golden["data_ty"]) and np.array_equal(cy, golden["data_cy"])
    assert np.abs(tx - golden["data_tx"]).max() < 1e-12
    assert np.abs(cx - golden["data_cx"]).max() < 1e-12


def test_init_random_bit_exact(golden):
    dims = [int(d) for d in golden["dims"]]
    assert np.array_equal(O.flatten(O.init_random(dims, 0, O.Rng(3))), golden["init_p0"])


def test_forward_backward(golden):
    dims = [int(d) for d in golden["dims"]]
    m = O.unflatten(golden["init_p0"], dims)
    x, y = golden["data_tx"][:24], golden["data_ty"][:24]
    tr = O.forward(m, x)
    assert np.abs(tr.z[-1] - golden["fwd_zlast"]).max() < 1e-12
    assert np.allclose(tr.a[-1].sum(axis=1), 1.0, atol=1e-12)  # SPEC: softmax rows sum to 1
    assert abs(O.cross_entropy(tr, y) - float(golden["fwd_ce"])) < 1e-12
    gW, gb, dzs = O.backward(m, tr, y, want_dz=True)
    flat = np.concatenate([np.concatenate([w.ravel(), b]) for w, b in zip(gW, gb)])
    assert np.abs(flat - golden["bwd_grads"]).max() < 1e-12
    for l, d in enumerate(dzs):
        assert np.abs(d - golden[f"bwd_dz{l}"]).max() < 1e-12


def test_finite_difference_gradient():
    # SPEC acceptance: FD gradient check on a 5-8-4-3 net (< 1e-6)
    dims = [5, 8, 4, 3]
    m = O.init_random(dims, 0, O.Rng(1))
    x = np.random.default_rng(0).standard_normal((6, 5))
    y = np.array([0, 1, 2, 0, 1, 2])
    gW, gb = O.backward(m, O.forward(m, x), y)
    eps = 1e-6
    for l in range(3):
        for (i, j) in [(0, 0), (1, 2), (dims[l + 1] - 1, dims[l] - 1)]:
            mp, mm = m.copy(), m.copy()
            mp.W[l][i, j] += eps
            mm.W[l][i, j] -= eps
            fd = (O.cross_entropy(O.forward(mp, x), y) - O.cross_entropy(O.forward(mm, x), y)) / (2 * eps)
            assert abs(fd - gW[l][i, j]) < 1e-6


def _replay(golden, ng):
    dims = [int(d) for d in golden["dims"]]
    m = O.unflatten(golden["init_p0"], dims)
    st = O.ng_init(m)
    x, y = golden["data_tx"], golden["data_ty"]
    rows = golden["steps_rows"].astype(np.int64)
    ces = []
    for s, lr in enumerate(golden["steps_lrs"]):
        rr = rows[s * 16:(s + 1) * 16]
        tr = O.forward(m, x[rr])
        ces.append(O.cross_entropy(tr, y[rr]))
        if ng:
            gW, gb, dzs = O.backward(m, tr, y[rr], want_dz=True)
            O.ng_update_state(st, tr, dzs)
            gW, gb = O.ng_precondition(st, gW, gb)
        else:
            gW, gb = O.backward(m, tr, y[rr])
        O.sgd_step(m, gW, gb, lr)
    return m, st, np.array(ces)


def test_one_averaging_period_sgd_and_ng(golden):
    for name, ng in (("sgd", False), ("ng", True)):
        m, st, ces = _replay(golden, ng)
        assert np.abs(O.flatten(m) - golden[f"steps_{name}_p"]).max() < 1e-11
        assert np.abs(ces - golden[f"steps_{name}_ce"]).max() < 1e-11
        if ng:
            for l in range(3):
                assert np.abs(st.r_in[l] - golden[f"steps_ng_rin{l}"]).max() < 1e-11
                assert np.abs(st.r_out[l] - golden[f"steps_ng_rout{l}"]).max() < 1e-11


def test_ng_invariants():
    # cold start == identity; norm preservation; diag example
    rng = np.random.default_rng(3)
    g = rng.standard_normal((4, 3))
    st = O.NgState([np.zeros((3, 3))], [np.zeros((4, 4))], [0])
    oW, ob = O.ng_precondition(st, [g], [np.ones(4)])
    assert np.abs(oW[0] - g).max() < 1e-9 and np.abs(ob[0] - 1.0).max() < 1e-9
    a = rng.standard_normal((10, 3))
    st2 = O.NgState([a.T @ a / 10], [np.eye(4) * 0.3], [1])
    oW, _ = O.ng_precondition(st2, [g], [np.ones(4)])
    assert abs(np.linalg.norm(oW[0]) - np.linalg.norm(g)) < 1e-9
    # hand case: S_in = diag(1,4), S_out = I, G = [[1,1]] -> Ghat = [[1,0.25]]
    gh = O.sandwich_solve(np.eye(1), np.array([[1.0, 1.0]]), np.diag([1.0, 4.0]))
    assert np.allclose(gh, [[1.0, 0.25]])


def test_allreduce(golden):
    assert np.array_equal(O.allreduce_average([np.array([1.0, 3.0]), np.array([3.0, 5.0])], 2), [2.0, 4.0])
    assert np.array_equal(O.allreduce_average(list(golden["avg_m7_in"]), 7), golden["avg_m7"])
    v = np.random.default_rng(1).standard_normal(9)
    assert np.array_equal(O.allreduce_average([v] * 4, 4), v)  # identical inputs -> bitwise fixed point
    for m in (1, 2, 3, 4, 7, 8, 16, 32):
        vs = list(np.random.default_rng(m).standard_normal((m, 17)))
        assert np.abs(O.allreduce_average(vs, m) - np.mean(vs, axis=0)).max() < 1e-12


def test_train_loop_matches_reference(golden):
    dims = [int(d) for d in golden["dims"]]
    m0 = O.unflatten(golden["init_p0"], dims)
    args = (golden["data_tx"], golden["data_ty"], golden["data_cx"], golden["data_cy"])
    for name, kw in (("tp_sgd_m4", dict(workers=4, avg_frequency=2, minibatch=8, ngsgd=False, epochs=3, lr_init=0.5)),
                     ("tp_ng_m2", dict(workers=2, avg_frequency=3, minibatch=8, ngsgd=True, epochs=2)),
                     ("tp_sgd_newbob_m2", dict(workers=2, avg_frequency=4, minibatch=8, ngsgd=False, newbob=True,
                                               epochs=4, lr_init=0.5))):
        m, met = O.train_loop(m0, *args, base_seed=17, **kw)
        ref = golden[f"{name}_met"]
        assert len(met) == ref.shape[0]
        assert np.abs(O.flatten(m) - golden[f"{name}_p"]).max() < 1e-10
        for e, mt in enumerate(met):
            assert mt.epoch == ref[e, 0] and abs(mt.lr - ref[e, 1]) < 1e-15
            assert abs(mt.train_ce - ref[e, 2]) < 1e-10 and abs(mt.cv_accuracy - ref[e, 3]) < 1e-12
            assert mt.workers == ref[e, 5] and mt.avg_events == ref[e, 6]


def test_schedules(golden):
    s = O.make_schedule(True, 0.32, 15)
    out = [O.newbob_next(s, a, b) for a, b in zip(golden["newbob_accs"][:-1], golden["newbob_accs"][1:])]
    assert np.allclose([o[0] for o in out], golden["newbob_lr"])
    assert [o[1] for o in out] == list(golden["newbob_stop"].astype(bool))
    e = O.make_schedule(False, 0.32, 15)
    assert np.allclose([O.exponential_lr(e, p) for p in (0.0, 0.5, 1.0, 0.25)], golden["explr"], rtol=0, atol=1e-17)
    assert abs(O.exponential_lr(e, 0.5) - 0.032) < 1e-15 and abs(O.exponential_lr(e, 1.0) - 0.0032) < 1e-15
    assert O.scale_lr_for_workers(0.32, 16) == pytest.approx(5.12) and O.scale_lr_for_workers(0.32, 32) == pytest.approx(10.24)
    # SPEC.md:253-255
    s = O.make_schedule(True, 0.32, 15)
    assert O.newbob_next(s, 0.5, 0.52) == (0.32, False)
    assert O.newbob_next(s, 0.52, 0.524)[0] == 0.16 and s.halving_active
    assert O.newbob_next(s, 0.524, 0.5245)[1]


def test_rbm_cd1(golden):
    for kind, gauss in (("bern", False), ("gauss", True)):
        p0 = golden[f"rbm_{kind}_p0"]
        v, h = 6, 4
        r = O.Rbm(p0[:h * v].reshape(h, v).copy(), p0[h * v:h * v + v].copy(), p0[h * v + v:].copy(), gauss)
        batch = golden[f"rbm_{kind}_batch"]
        pos, hs, rec, neg = O.cd1_gibbs(r, batch, O.threshold_half)
        out = O.cd1_apply(r, batch, pos, rec, neg, 0.1)
        flat = np.concatenate([out.W.ravel(), out.vb, out.hb])
        assert np.abs(flat - golden[f"rbm_{kind}_thr_p"]).max() < 1e-12
        rng = O.Rng(99)
        pos, hs, rec, neg = O.cd1_gibbs(r, batch, lambda p: O.sample_bernoulli(p, rng))
        assert np.array_equal(hs, golden[f"rbm_{kind}_rng_hs"])
        out = O.cd1_apply(r, batch, pos, rec, neg, 0.1)
        assert np.abs(np.concatenate([out.W.ravel(), out.vb, out.hb]) - golden[f"rbm_{kind}_rng_p"]).max() < 1e-12
        assert abs(O.reconstruction_error(r, batch) - float(golden[f"rbm_{kind}_recerr"])) < 1e-12


def test_cd1_hand_case():
    # lr = 0 leaves parameters unchanged; identical data/recon stats -> zero update
    r = O.Rbm(np.array([[0.5, -0.5]]), np.zeros(2), np.zeros(1), False)
    v = np.array([[1.0, 0.0]])
    pos, hs, rec, neg = O.cd1_gibbs(r, v, O.threshold_half)
    same = O.cd1_apply(r, v, pos, rec, neg, 0.0)
    assert np.array_equal(same.W, r.W)
    z = O.cd1_apply(r, v, pos, v, pos, 0.7)
    assert np.allclose(z.W, r.W) and np.allclose(z.hb, r.hb)


def test_greedy_pretrain(golden):
    dims = [int(d) for d in golden["pre_dims"]]
    m = O.greedy_pretrain(dims, golden["data_tx"][:64], O.Rng(41), epochs=2, batch=8)
    assert np.abs(O.flatten(m) - golden["pre_p"]).max() < 1e-10


def test_checkpoint_bytes(golden):
    dims = [int(d) for d in golden["dims"]]
    m = O.unflatten(golden["init_p0"], dims)
    buf = O.save_model_bytes(m)
    assert buf == golden["ckpt_bytes"].tobytes()
    back = O.load_model_bytes(buf)
    assert np.array_equal(O.flatten(back), golden["init_p0"])
    with pytest.raises(ValueError, match="bad magic"):
        O.load_model_bytes(b"XXXXXXXX" + buf[8:])


def test_live_reference_agrees(reflib):
    # When the compiled reference is present, cross-check a fresh random case.
    dims = [9, 7, 5]
    p = reflib.init_random(dims, 123)
    assert np.array_equal(p, O.flatten(O.init_random(dims, 0, O.Rng(123))))
    x = np.random.default_rng(4).standard_normal((11, 9))
    y = np.arange(11) % 5
    _, _, ce = reflib.forward(dims, p, x, y)
    assert abs(ce - O.cross_entropy(O.forward(O.unflatten(p, dims), x), y)) < 1e-12
    assert math.isfinite(reflib.time_ng_precondition(16, 12))


@pytest.mark.parametrize("ngsgd", [False, True])
def test_threaded_reference_step_equals_reference(reflib, ngsgd):
    """bench.py's reference arm (one true-width step of the reference's own
    functions spread over host threads, ref_time_step_threaded) computes the
    reference's single-threaded step (ref_train_steps) up to fp64 summation
    order, including an output layer wide enough (rows > 2 x columns) to take
    the column-chunked solves."""
    dims = [40, 64, 48, 1100]
    B = 96
    rng = np.random.default_rng(0)
    x = rng.standard_normal((B, dims[0]))
    y = rng.integers(0, dims[-1], B).astype(np.int32)
    p0 = reflib.init_random(dims, 3)
    wall, ph, p, ce = reflib.time_step_threaded(dims, p0, x, y, ngsgd, 5, lr=0.3)
    pr, cer, _, _ = reflib.train_steps(dims, p0, x, y, np.arange(B), B, [0.3], ngsgd)
    assert wall > 0 and np.all(ph >= 0)
    assert np.abs(p - pr).max() <= 1e-9 * np.abs(pr - p0).max()
    assert abs(ce - cer[0]) <= 1e-12 * abs(cer[0])


def test_oracle_config1_period_matches_reference_digest():
    """The numpy oracle is pinned at the config-1 shape too (440-512-512-1000,
    batch 256): one averaging period from the reference's own fixture."""
    import os
    from conftest import ROOT
    from paper_1507_01239_b200 import parnn as P
    g = dict(np.load(os.path.join(ROOT, "tests", "golden", "golden_cfg1.npz")))
    dims = [440, 512, 512, 1000]
    tr, _ = P.make_data(1000, 440, 100, float(g["separation"]), 7, 0.10, 2, True)
    m = O.unflatten(P.init_random(dims, seed=1).params, dims)
    rows = P.minibatch_rows(tr.size(), 256, 21)[:4].ravel().astype(np.int64)
    ces = []
    for s, lr in enumerate([0.32, 0.3, 0.28, 0.26]):
        rr = rows[s * 256:(s + 1) * 256]
        t = O.forward(m, tr.features[rr])
        ces.append(O.cross_entropy(t, tr.labels[rr]))
        gW, gb = O.backward(m, t, tr.labels[rr])
        O.sgd_step(m, gW, gb, lr)
    p = O.flatten(m)
    assert rel(p[g["digest_idx"]], g["period_p_digest"]) < 1e-12
    assert np.abs(np.array(ces) - g["period_ce"]).max() < 1e-12
