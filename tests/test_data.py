"""Data ingress: load_csv / save_csv against the compiled
reference (data.cpp:66-122) -- the same rows, labels and classes, and the same
error message (text and 1-based line) for every malformed input -- and, on the
GPU, the device-side generate_synthetic + split_cv + standardize against the
host restatement (labels / row order bit-exact, features within fp32
rounding)."""
import os

import numpy as np
import pytest

from paper_1507_01239_b200 import parnn as P

CASES = {
    "ok_spaces": " 2 , 3.5 ,\t4 \r\n# comment\n\n0,1e-3,-2\n1,0x10,+7\n",
    "one_field": "1\n",
    "bad_label": "a,1,2\n",
    "neg_label": "-1,1\n",
    "frac_label": "1.5,2\n",
    "ragged": "1,2,3\n1,2\n",
    "bad_feature": "1,2,x\n",
    "nan_feature": "1,nan\n",
    "range_feature": "1,1e999\n",
    "trailing_junk": "1,2.5abc\n",
    "only_comments": "# nothing\n\n   \n",
    "empty_field": "1,,2\n",
    "no_newline_end": "3,1,2\n4,5,6",
}


def _write(tmp_path, name, text):
    p = tmp_path / f"{name}.csv"
    p.write_bytes(text.encode())
    return str(p)


def _both(reflib, path):
    """(ours, reference): each either (x, y, classes) or ('error', message)."""
    out = []
    for f in (lambda: P.load_csv(path), lambda: reflib.load_csv(path)):
        try:
            r = f()
            out.append((r.features, r.labels, r.num_classes) if isinstance(r, P.Dataset) else r)
        except (P.ParnnError, RuntimeError) as e:
            out.append(("error", str(e)))
    return out


@pytest.mark.parametrize("name", sorted(CASES))
def test_load_csv_matches_reference(reflib, tmp_path, name):
    ours, ref = _both(reflib, _write(tmp_path, name, CASES[name]))
    if isinstance(ref[0], str):
        assert isinstance(ours[0], str) and ours[1] == ref[1]
    else:
        assert np.array_equal(ours[0], ref[0]) and np.array_equal(ours[1], ref[1]) and ours[2] == ref[2]


def test_load_csv_missing_file(reflib, tmp_path):
    ours, ref = _both(reflib, str(tmp_path / "nope.csv"))
    assert ours == ref and isinstance(ref[0], str)


@pytest.mark.parametrize("where", ["none", "early", "chunk_boundary", "late"])
def test_load_csv_large_threaded(reflib, tmp_path, where):
    """A file large enough to be parsed in many chunks: the first error in file
    order wins, a ragged row is judged against the file's first row."""
    rng = np.random.default_rng(0)
    n, d = 60000, 6
    x = rng.standard_normal((n, d))
    y = rng.integers(0, 17, n).astype(np.int32)
    lines = [",".join([str(int(y[i]))] + ["%.17g" % v for v in x[i]]) for i in range(n)]
    if where == "early":
        lines[12] = lines[12] + ",3"  # ragged vs the first row
        lines[40000] = "x,1,2,3,4,5,6"
    elif where == "chunk_boundary":
        lines[n // 2] = lines[n // 2].rsplit(",", 1)[0]  # one feature short
    elif where == "late":
        lines[n - 3] = lines[n - 3].replace(",", ",q", 1)
    path = _write(tmp_path, f"big_{where}", "\n".join(lines) + "\n")
    ours, ref = _both(reflib, path)
    if isinstance(ref[0], str):
        assert ours == ref
    else:
        assert np.array_equal(ours[0], ref[0]) and np.array_equal(ours[1], ref[1]) and ours[2] == ref[2]


def test_save_csv_bytes_match_reference(reflib, tmp_path):
    rng = np.random.default_rng(1)
    ds = P.Dataset(rng.standard_normal((37, 5)) * 1e3, rng.integers(0, 4, 37).astype(np.int32), 4)
    a, b = str(tmp_path / "ours.csv"), str(tmp_path / "ref.csv")
    P.save_csv(a, ds)
    reflib.save_csv(b, ds.features, ds.labels)
    assert open(a, "rb").read() == open(b, "rb").read()
    back = P.load_csv(a)
    assert np.array_equal(back.features, ds.features) and np.array_equal(back.labels, ds.labels)


@pytest.mark.gpu
@pytest.mark.parametrize("shape", [(50, 37, 7, 3.0, 11, 2), (1000, 440, 20, 16.0, 7, 2), (8806, 440, 3, 8.0, 1, 2)])
def test_device_generate_matches_host(ctx, shape):
    classes, dim, per_class, sep, seed, split_seed = shape
    tr, cv = P.make_data(classes, dim, per_class, sep, seed, 0.10, split_seed, True)
    dtr, dcv = P.DeviceDataset.generate(ctx, classes, dim, per_class, sep, seed, 0.10, split_seed, True)
    for host, dev in ((tr, dtr.download()), (cv, dcv.download())):
        assert dev.features.shape == host.features.shape
        assert np.array_equal(dev.labels, host.labels)  # class order + split permutation: bit-exact
        err = np.abs(dev.features.astype(np.float64) - host.features)
        assert err.max() <= 2e-6 * max(1.0, np.abs(host.features).max())  # fp32 rounding of the fp64 values
    # unstandardized too (the raw mean + noise values)
    tr0, _ = P.make_data(classes, dim, per_class, sep, seed, 0.10, split_seed, False)
    d0, _ = P.DeviceDataset.generate(ctx, classes, dim, per_class, sep, seed, 0.10, split_seed, False)
    assert np.abs(d0.download().features - tr0.features).max() <= 2e-6 * np.abs(tr0.features).max()


@pytest.mark.gpu
def test_device_generate_trains_like_host(ctx):
    """A device-generated set is a drop-in for the host one: the same
    train_parallel run on either gives the same metrics (fp32 mode)."""
    dims = [24, 32, 10]
    tr, cv = P.make_data(10, 24, 30, 4.0, 3, 0.10, 5, True)
    dtr, dcv = P.DeviceDataset.generate(ctx, 10, 24, 30, 4.0, 3, 0.10, 5, True)
    m0 = P.init_random(dims, seed=2)
    opts = P.TrainOptions(optimizer=P.OptimizerKind.sgd, lr_init=0.5, epochs=2, precision=P.Precision.fp32)
    plan = P.ParallelPlan(2, 2, 8, 3)
    a = P.train_parallel(plan, m0, tr, cv, opts, ctx=ctx)
    b = P.train_parallel(plan, m0, tr, cv, opts, ctx=ctx, device_data=(dtr, dcv))
    for x, y in zip(a.metrics, b.metrics):
        assert abs(x.train_ce - y.train_ce) <= 1e-5 * x.train_ce and abs(x.cv_accuracy - y.cv_accuracy) <= 0.02


@pytest.mark.gpu
def test_dataset_load_csv_device(ctx, tmp_path):
    rng = np.random.default_rng(2)
    ds = P.Dataset(rng.standard_normal((100, 9)), rng.integers(0, 5, 100).astype(np.int32), 5)
    path = str(tmp_path / "d.csv")
    P.save_csv(path, ds)
    dd = P.DeviceDataset.load_csv(ctx, path)
    back = dd.download()
    assert dd.num_classes == int(ds.labels.max()) + 1
    assert np.array_equal(back.labels, ds.labels)
    assert np.array_equal(back.features, ds.features.astype(np.float32))


@pytest.mark.parametrize("args", [(0, 5, 3, 2.0, 1, 0.1, 2), (3, 5, 3, 2.0, 1, 1.0, 2), (3, 5, 3, 2.0, 1, 0.0, 2),
                                  (3, 5, 3, -1.5, 1, 0.1, 2), (3, 5, 3, 2.0, 1, -1e-9, 2), (2, 4, 1, 2.0, 1, 0.5, 2)])
def test_generate_errors_match_reference(reflib, args):
    """generate_synthetic / split_cv validation (data.cpp:124-183): the same
    message, doubles formatted as the reference's operator<< prints them."""
    msgs = []
    for f in (lambda: reflib.make_data(*args, True), lambda: P.make_data(*args, True)):
        with pytest.raises((RuntimeError, P.ParnnError)) as e:
            f()
        msgs.append(str(e.value))
    assert msgs[0] == msgs[1]


def test_schedule_errors_match_reference(reflib):
    """LR schedule validation (optimizer.cpp:159-208), the same text incl. the
    values: newbob against the compiled reference; exponential_lr /
    make_schedule against the reference's literal messages (its shim returns a
    value instead of raising)."""
    msgs = []
    for lib in (reflib, P):
        with pytest.raises((RuntimeError, P.ParnnError)) as e:
            lib.newbob_sequence(0.32, [0.5, 1.2])
        msgs.append(str(e.value))
    assert msgs[0] == msgs[1] == "newbob_next: accuracies must be in [0,1], got 0.5 and 1.2"
    with pytest.raises(P.ParnnError, match=r"^exponential_lr: progress must be in \[0,1\], got 1\.5$"):
        P.exponential_lr(0.32, 5, 1.5)
    with pytest.raises(P.ParnnError, match=r"^make_schedule: lr_init must be positive, got -0\.25$"):
        P.exponential_lr(-0.25, 5, 0.5)
