"""Config 1 with the reference's own kron-full NG-SGD on the compiled reference
-- the pin for this framework's kron-full NG over whole runs and the baseline
for the low-rank NG-SGD update-lag comparison.

    make -C oracle && python tests/golden/make_golden_cfg1_ng.py [full|small|both]

* golden_cfg1_ng.npz: 100 frames per class, 2 epochs (about 23 minutes on one
  core) -- per-epoch EpochMetrics.
* golden_cfg1_ng_small.npz: 10 frames per class (9000 train frames, 35 steps),
  1 epoch (about 70 s) -- EpochMetrics plus 64 Rademacher projections of the
  parameter delta (a compact fingerprint of the whole trajectory: the test
  projects its own delta with the same matrix, rng_projection below).
Both: 440-512-512-1000 sigmoid, 1 worker, averaging period 4, minibatch 256,
base seed 5, exponential schedule from lr 2.0, decay 0.95, smoothing 4."""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle.ref_lib import RefLib  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
DIMS = [440, 512, 512, 1000]
SEPARATION, LR_INIT = 16.0, 2.0


def rng_projection(n, k=64, seed=0):
    """k x n Rademacher matrix (float32), applied in row blocks to bound memory."""
    return np.random.default_rng(seed).integers(0, 2, (k, n), dtype=np.int8).astype(np.float32) * 2 - 1


def run(R, per_class, epochs):
    (tx, ty), (cx, cy) = R.make_data(1000, 440, per_class, SEPARATION, 7, 0.1, 2, True)
    p0 = R.init_random(DIMS, 1)
    t0 = time.time()
    p, met = R.train_parallel(DIMS, p0, tx, ty, cx, cy, workers=1, avg_frequency=4, minibatch=256, base_seed=5,
                              ngsgd=True, lr_init=LR_INIT, epochs=epochs)
    return p0, p, met, time.time() - t0


def main():
    which = sys.argv[1] if len(sys.argv) > 1 else "both"
    R = RefLib()
    if which in ("full", "both"):
        _, _, met, wall = run(R, 100, 2)
        out = os.path.join(HERE, "golden_cfg1_ng.npz")
        np.savez_compressed(out, met=met, separation=np.array(SEPARATION), lr_init=np.array(LR_INIT),
                            epochs=np.array(2), wall_seconds=np.array(wall))
        print("wrote", out, met[:, 2], met[:, 3], wall)
    if which in ("small", "both"):
        p0, p, met, wall = run(R, 10, 1)
        d = (p - p0).astype(np.float32)
        proj = rng_projection(d.size) @ d
        out = os.path.join(HERE, "golden_cfg1_ng_small.npz")
        np.savez_compressed(out, met=met, proj=proj, delta_norm=np.array(np.linalg.norm(p - p0)),
                            params_norm=np.array(np.linalg.norm(p)), wall_seconds=np.array(wall))
        print("wrote", out, met, wall)


if __name__ == "__main__":
    main()
