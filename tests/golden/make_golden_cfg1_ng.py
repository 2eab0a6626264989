"""Config 1 with the reference's own kron-full NG-SGD (2 epochs) on the compiled
reference -- the baseline for the low-rank NG-SGD update-lag comparison
(lag 1 and lag 4 must reach the reference's NG CE within 1%).
About 20 minutes on one core:
    make -C oracle && python tests/golden/make_golden_cfg1_ng.py
Writes tests/golden/golden_cfg1_ng.npz (per-epoch EpochMetrics)."""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle.ref_lib import RefLib  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden_cfg1_ng.npz")
DIMS = [440, 512, 512, 1000]
SEPARATION, LR_INIT, EPOCHS = 16.0, 2.0, 2


def main():
    R = RefLib()
    (tx, ty), (cx, cy) = R.make_data(1000, 440, 100, SEPARATION, 7, 0.1, 2, True)
    p0 = R.init_random(DIMS, 1)
    t0 = time.time()
    _, met = R.train_parallel(DIMS, p0, tx, ty, cx, cy, workers=1, avg_frequency=4, minibatch=256, base_seed=5,
                              ngsgd=True, lr_init=LR_INIT, epochs=EPOCHS)
    np.savez_compressed(OUT, met=met, separation=np.array(SEPARATION), lr_init=np.array(LR_INIT),
                        epochs=np.array(EPOCHS), wall_seconds=np.array(time.time() - t0))
    print("wrote", OUT, met[:, 2], met[:, 3], time.time() - t0)


if __name__ == "__main__":
    main()
