"""CD-1 throughput of greedy_pretrain at config-4 layer shapes (pretrain.cpp:162-207):
440->2048 (Gaussian-Bernoulli) and 2048->2048, batch 128, on N synthetic frames.
Prints one line per precision: seconds, steps, us/step, TFLOP/s (10 v h flop per
frame per RBM).

    python scripts/cd1_time.py [n_frames] [epochs] [dims]
"""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1507_01239_b200 import parnn as P  # noqa: E402


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 65536
    epochs = int(sys.argv[2]) if len(sys.argv) > 2 else 2
    dims = [int(x) for x in sys.argv[3].split(",")] if len(sys.argv) > 3 else [440, 2048, 2048, 2048, 10]
    x = np.random.default_rng(0).standard_normal((n, dims[0]))
    ctx = P.Context(0)
    rbms = list(zip(dims[:-2], dims[1:-1]))
    for prec in (P.Precision.tf32, P.Precision.bf16, P.Precision.fp32):
        P.greedy_pretrain(dims, x[:4096], P.PretrainOptions(1), seed=1, precision=prec, ctx=ctx)  # warm-up
        t0 = time.perf_counter()
        P.greedy_pretrain(dims, x, P.PretrainOptions(epochs), seed=2, precision=prec, ctx=ctx)
        wall = time.perf_counter() - t0
        st = P.pretrain_last_stats()
        us = st["cd1_device_seconds"] / st["cd1_steps"] * 1e6
        print(f"{prec.name:5s} dims={'-'.join(map(str, dims))} n={n} epochs={epochs}: {st['cd1_steps']} CD-1 steps, "
              f"device {st['cd1_device_seconds']:.4f} s = {us:.1f} us/step, "
              f"{st['cd1_flop'] / st['cd1_device_seconds'] / 1e12:.1f} TFLOP/s (call wall {wall:.3f} s)", flush=True)


if __name__ == "__main__":
    main()
