"""Generate tests/golden/golden_cfg1.npz: BASELINE.json config 1 on the
UNMODIFIED reference compiled by oracle/Makefile (oracle/_ref). Run where
/root/reference exists (about 10 minutes on one core):

    make -C oracle && python tests/golden/make_golden_cfg1.py

Config 1: 440-512-512-1000 sigmoid, plain SGD, one worker, minibatch 256,
100k synthetic frames (generate_synthetic(1000, 440, 100, s, seed 7), split_cv
0.1 seed 2, standardized). The separation s = 16 and lr_init = 2.0 were chosen
with the numpy oracle so that the cross-entropy falls well below ln 1000 within
the 4 epochs (SURVEY §8d "Calibrate s"; at s = 3 / lr 0.32 it stays at ln 1000):
the per-epoch CE gate then compares a trajectory that actually moves.

Stored: the per-epoch EpochMetrics of train_parallel, and a digest of the
parameters (10^4 fixed coordinates) after the full run and after one
averaging period (4 steps, batch 256) from the initial model, plus the
per-step CE of that period.
"""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle.ref_lib import RefLib  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden_cfg1.npz")
DIMS = [440, 512, 512, 1000]
SEPARATION, LR_INIT, EPOCHS = 16.0, 2.0, 4


def main():
    R = RefLib()
    (tx, ty), (cx, cy) = R.make_data(1000, 440, 100, SEPARATION, 7, 0.1, 2, True)
    p0 = R.init_random(DIMS, 1)
    P = R.param_count(DIMS)
    idx = np.sort(np.random.default_rng(2024).choice(P, 10000, replace=False)).astype(np.int64)
    g = {"separation": np.array(SEPARATION), "lr_init": np.array(LR_INIT), "epochs": np.array(EPOCHS),
         "digest_idx": idx}
    # one averaging period (K = 4 steps) from the initial model
    rows = R.minibatch_rows(tx.shape[0], 256, 21)[:4].ravel()
    lrs = [0.32, 0.3, 0.28, 0.26]
    p4, ce4, _, _ = R.train_steps(DIMS, p0, tx, ty, rows, 256, lrs, False)
    g["period_p_digest"], g["period_ce"] = p4[idx], ce4
    # the full run (train_parallel, one worker, averaging every 4)
    t0 = time.time()
    p, met = R.train_parallel(DIMS, p0, tx, ty, cx, cy, workers=1, avg_frequency=4, minibatch=256, base_seed=5,
                              ngsgd=False, lr_init=LR_INIT, epochs=EPOCHS)
    g["met"], g["final_p_digest"] = met, p[idx]
    g["wall_seconds"] = np.array(time.time() - t0)
    np.savez_compressed(OUT, **g)
    print("wrote", OUT, os.path.getsize(OUT), "bytes;", met[:, 2], met[:, 3], "wall", time.time() - t0)


if __name__ == "__main__":
    main()
