"""Config 4: RBM CD-1 greedy pretraining of the 6x2048 stack (Gaussian-
Bernoulli first layer), then NG-SGD fine-tuning (BASELINE.json configs[3];
SURVEY §8(a) A15, §8(d) cfg4).

1. ``greedy_pretrain`` (pretrain.cpp:162-207) on the standardized synthetic
   train frames with the reference's PretrainOptions (batch 128, lr 0.001
   Gaussian / 0.1 Bernoulli), timed with the device synchronised on both
   sides; CD-1 throughput = frames x epochs x layers / time, against
   10 d_v d_h flop per frame per layer.
2. Fine-tune with ``train_parallel`` (low-rank NG-SGD, minibatch 1024,
   averaging every 4) from the pretrained stack and from ``init_random``:
   per-epoch train CE and CV accuracy of both.
3. Reference CPU CD-1 (oracle/_ref, 1 thread): one step per layer shape, as a
   bounded sample (``--no-cpu`` skips it).

One GPU: the replicas of a multi-GPU fine-tune are independent between
averaging events, so one GPU's share is this run with workers / GPUs.
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_1507_01239_b200 import parnn as P  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--per-class", type=int, default=24)
    ap.add_argument("--pretrain-epochs", type=int, default=10)
    ap.add_argument("--finetune-epochs", type=int, default=3)
    ap.add_argument("--precision", choices=["bf16", "tf32", "fp32"], default="tf32")
    ap.add_argument("--workers", type=int, default=1)
    ap.add_argument("--lr-init", type=float, default=0.32)
    ap.add_argument("--separation", type=float, default=8.0)
    ap.add_argument("--dims", default="440,2048,2048,2048,2048,2048,2048,8806")
    ap.add_argument("--no-cpu", action="store_true")
    args = ap.parse_args()
    dims = [int(x) for x in args.dims.split(",")]
    prec = P.Precision[args.precision]

    t0 = time.perf_counter()
    train, cv = P.make_data(dims[-1], dims[0], args.per_class, args.separation, 1, 0.10, 2, True)
    gen_s = time.perf_counter() - t0
    ctx = P.Context(0)
    opts = P.PretrainOptions()
    opts.epochs = args.pretrain_epochs
    # warm-up: one epoch of the first layer pair on a slice (JIT-free, but allocs / first launches)
    P.greedy_pretrain(dims[:3], train.features[:1024], P.PretrainOptions(1), seed=3, precision=prec, ctx=ctx)
    t0 = time.perf_counter()
    pre = P.greedy_pretrain(dims, train.features, opts, seed=11, precision=prec, ctx=ctx)
    pre_s = time.perf_counter() - t0
    cd1_st = P.pretrain_last_stats()
    n = train.size()
    n_eff = n // opts.batch_size * opts.batch_size
    rbm_layers = list(zip(dims[:-2], dims[1:-1]))
    flop = sum(10.0 * v * h for v, h in rbm_layers) * n_eff * opts.epochs
    out = {
        "workload": f"config 4: greedy_pretrain {'-'.join(map(str, dims[:-1]))} on {n} frames x {opts.epochs} epochs "
                    f"(batch {opts.batch_size}, {args.precision}), then low-rank NG-SGD fine-tune",
        "data_gen_seconds": gen_s,
        "pretrain_seconds": pre_s,
        "pretrain_frames_per_s_per_layer": n_eff * opts.epochs * len(rbm_layers) / pre_s,
        "pretrain_tflops": flop / pre_s / 1e12,
        "pretrain_flop_note": "10 d_v d_h flop per frame per RBM (SURVEY 8(d))",
        "pretrain_cd1_device_seconds": cd1_st["cd1_device_seconds"],
        "pretrain_cd1_tflops_device": cd1_st["cd1_flop"] / cd1_st["cd1_device_seconds"] / 1e12,
        "pretrain_cd1_us_per_step": cd1_st["cd1_device_seconds"] / cd1_st["cd1_steps"] * 1e6,
        "separation": args.separation, "lr_init": args.lr_init,
    }

    topts = P.TrainOptions(optimizer=P.OptimizerKind.ngsgd_lowrank, lr_schedule=P.LrVariant.exponential,
                           lr_init=args.lr_init, epochs=args.finetune_epochs, precision=P.Precision.bf16)
    plan = P.ParallelPlan(args.workers, 4, 1024, 0)
    for name, m0 in (("pretrained", pre), ("random_init", P.init_random(dims, seed=7))):
        res = P.train_parallel(plan, m0, train, cv, topts, ctx=ctx)
        out[f"finetune_{name}"] = [{"epoch": m.epoch, "train_ce": m.train_ce, "cv_accuracy": m.cv_accuracy,
                                    "wall_seconds": m.wall_seconds} for m in res.metrics]

    if not args.no_cpu:
        from oracle import ref_lib
        if ref_lib.available():
            ref = ref_lib.RefLib()
            rng = np.random.default_rng(0)
            cpu = {}
            for v, h, g in ((dims[0], dims[1], True), (dims[1], dims[2], False)):
                p = ref.rbm_init(v, h, g, 5)
                x = train.features[:opts.batch_size, :v] if v == dims[0] else rng.random((opts.batch_size, v))
                t0 = time.perf_counter()
                ref.cd1_update(v, h, g, p, x, 0.001 if g else 0.1, 0, 1)
                dt = time.perf_counter() - t0
                cpu[f"{v}x{h}"] = {"seconds_per_step": dt, "frames_per_s": opts.batch_size / dt}
            total = sum(opts.batch_size / cpu[f"{v}x{h}"]["frames_per_s"] if f"{v}x{h}" in cpu else
                        opts.batch_size / cpu[f"{dims[1]}x{dims[2]}"]["frames_per_s"] for v, h in rbm_layers)
            out["cpu_baseline"] = {"kind": "reference", "cores": 1, "per_shape": cpu,
                                   "frames_per_s_per_layer": opts.batch_size * len(rbm_layers) / total,
                                   "sample": "one reference cd1_update step (batch 128) per RBM shape"}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
