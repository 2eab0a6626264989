"""Probe the device eigensolver through parnn_debug_lowrank_eig on Z = K."""
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import ng_lowrank as LR  # noqa: E402
from paper_1507_01239_b200._lib import check, lib, ptr  # noqa: E402

for R in [20, 40, 64, 66, 72, 80, 96]:
    rng = np.random.default_rng(0)
    A = rng.standard_normal((R, 3 * R))
    K = (A @ A.T / (3 * R)).astype(np.float32)
    gram = np.zeros((2 * R, 2 * R), np.float32)
    gram[:R, :R] = K
    D = 4096
    st = np.zeros(2 * R + 12)
    st[:R] = 1.0
    st[R:2 * R] = 1.0
    st[2 * R] = 0.0
    st[2 * R + 1] = 1.0
    d1, rho1, e1, m = LR.eig_update(st[:R], st[R:2 * R], 0.0, K.astype(np.float64), np.zeros((R, R)), np.zeros((R, R)),
                                    1.0, D, 1.0, 1.0, 4.0)
    sout = np.zeros(2 * R + 12)
    mg = np.zeros((R, 2 * R), np.float32)
    sw = C.c_int()
    check(lib().parnn_debug_lowrank_eig(R, D, 1.0, 1.0, 4.0, ptr(st), ptr(gram), ptr(sout), ptr(mg), C.byref(sw)))
    ph = sout[2 * R + 5:2 * R + 10]
    rounds = sw.value * (((R + 7) // 8 * 8) // 4 - 1)
    print(R, "sweeps", sw.value, "d rel err", np.abs(sout[:R] - d1).max() / d1.max(), "cycles/round", round(sout[2 * R + 4] / max(rounds, 1)),
          "cycles", sout[2 * R + 4])
