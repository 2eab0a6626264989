"""Generate tests/golden/golden.npz from the UNMODIFIED reference compiled by
oracle/Makefile (oracle/_ref/libparnn_ref.so). Run in the survey container
(where /root/reference exists):

    make -C oracle && python tests/golden/make_golden.py

The fixtures pin both the numpy restatement (oracle/parnn_oracle.py) and the
CUDA path; they are small so they travel with the repo.
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle.ref_lib import RefLib  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden.npz")


def main():
    R = RefLib()
    g = {}
    # ---- rng / index streams (integer: bit-exact)
    g["rng_u64_s7"] = R.rng_u64(7, 64)
    g["rng_uniform_s11"] = R.rng_uniform(11, 64)
    g["rng_gauss_s3"] = R.rng_gaussian(3, 101)
    g["rng_index_s5_b10"] = R.rng_index(5, 10, 100)
    g["shuffle_1000_s5"] = R.shuffled_indices(1000, 5)
    g["partition_10_3_s9"] = R.partition_rows(10, 3, 9)
    g["partition_1000_7_s11"] = R.partition_rows(1000, 7, 11)
    g["minibatch_10_3_s11"] = R.minibatch_rows(10, 3, 11)
    g["minibatch_500_32_s13"] = R.minibatch_rows(500, 32, 13)
    # ---- data
    (tx, ty), (cx, cy) = R.make_data(10, 12, 20, 4.0, 1, 0.1, 2, True)
    g["data_tx"], g["data_ty"], g["data_cx"], g["data_cy"] = tx, ty, cx, cy
    # ---- model / forward / backward
    dims = [12, 16, 14, 10]
    g["dims"] = np.array(dims, np.uint64)
    p0 = R.init_random(dims, 3)
    g["init_p0"] = p0
    zs, as_, ce = R.forward(dims, p0, tx[:24], ty[:24])
    g["fwd_zlast"], g["fwd_alast"], g["fwd_ce"] = zs[-1], as_[-1], np.array(ce)
    grads, dz = R.backward(dims, p0, tx[:24], ty[:24])
    g["bwd_grads"] = grads
    for l, d in enumerate(dz):
        g[f"bwd_dz{l}"] = d
    # ---- one averaging period (K = 4 steps) for SGD and NG-SGD
    rows = R.minibatch_rows(tx.shape[0], 16, 21)[:4].ravel()
    lrs = [0.32, 0.28, 0.25, 0.2]
    g["steps_rows"], g["steps_lrs"] = rows, np.array(lrs)
    for name, ng in (("sgd", False), ("ng", True)):
        p, ces, fac, lastg = R.train_steps(dims, p0, tx, ty, rows, 16, lrs, ng)
        g[f"steps_{name}_p"], g[f"steps_{name}_ce"] = p, ces
        if ng:
            for l, (ri, ro) in enumerate(fac):
                g[f"steps_ng_rin{l}"], g[f"steps_ng_rout{l}"] = ri, ro
            g["steps_ng_lastgrad"] = lastg
    # ---- allreduce
    g["avg_m2"] = R.allreduce_average(np.array([[1.0, 3.0], [3.0, 5.0]]))
    rnd = np.random.default_rng(5).standard_normal((7, 33))
    g["avg_m7_in"], g["avg_m7"] = rnd, R.allreduce_average(rnd)
    # ---- full train loops (train_parallel / serial_train)
    runs = {
        "tp_sgd_m4": dict(workers=4, avg_frequency=2, minibatch=8, ngsgd=False, newbob=False, epochs=3, lr_init=0.5),
        "tp_ng_m2": dict(workers=2, avg_frequency=3, minibatch=8, ngsgd=True, newbob=False, epochs=2, lr_init=0.32),
        "tp_sgd_newbob_m2": dict(workers=2, avg_frequency=4, minibatch=8, ngsgd=False, newbob=True, epochs=4, lr_init=0.5),
        "serial_sgd": dict(workers=1, avg_frequency=1, minibatch=8, ngsgd=False, newbob=False, epochs=2, lr_init=0.5,
                           serial=True),
    }
    for name, kw in runs.items():
        p, met = R.train_parallel(dims, p0, tx, ty, cx, cy, base_seed=17, **kw)
        g[f"{name}_p"], g[f"{name}_met"] = p, met
    # ---- schedules
    accs = np.array([0.5, 0.52, 0.524, 0.528, 0.5285, 0.53])
    lr, st = R.newbob_sequence(0.32, accs)
    g["newbob_accs"], g["newbob_lr"], g["newbob_stop"] = accs, lr, st
    g["explr"] = np.array([R.exponential_lr(0.32, 15, p) for p in (0.0, 0.5, 1.0, 0.25)])
    # ---- RBM CD-1 (threshold stub and seeded sampling), reconstruction error
    for kind, gauss in (("bern", False), ("gauss", True)):
        v, h, b = 6, 4, 5
        rp = R.rbm_init(v, h, gauss, 31)
        batch = np.random.default_rng(7).random((b, v)) if not gauss else np.random.default_rng(7).standard_normal((b, v))
        out_t, tr_t = R.cd1_update(v, h, gauss, rp, batch, 0.1, 1)
        out_r, tr_r = R.cd1_update(v, h, gauss, rp, batch, 0.1, 0, seed=99)
        g[f"rbm_{kind}_p0"], g[f"rbm_{kind}_batch"] = rp, batch
        g[f"rbm_{kind}_thr_p"], g[f"rbm_{kind}_rng_p"] = out_t, out_r
        g[f"rbm_{kind}_rng_hs"] = tr_r[1]
        g[f"rbm_{kind}_recerr"] = np.array(R.reconstruction_error(v, h, gauss, rp, batch))
    pre_dims = [12, 10, 8, 10]
    g["pre_dims"] = np.array(pre_dims, np.uint64)
    g["pre_p"] = R.greedy_pretrain(pre_dims, tx[:64], 2, 0.001, 0.1, 8, 41)
    # ---- checkpoint bytes
    path = "/tmp/golden_model.bin"
    R.save_model(path, dims, p0)
    g["ckpt_bytes"] = np.frombuffer(open(path, "rb").read(), np.uint8)
    np.savez_compressed(OUT, **g)
    print("wrote", OUT, os.path.getsize(OUT), "bytes", len(g), "arrays")


if __name__ == "__main__":
    main()
