"""Config 5: averaging-frequency x minibatch sweep with virtual replicas
(BASELINE.json configs[4]).

Runs ``train_parallel`` (440-2048x6-8806 sigmoid, low-rank NG-SGD by default)
for every (minibatch, avg_frequency) cell with ``--workers`` replicas hosted
on this one GPU (the paper's 32-GPU setup is 32 workers; one B200 of the
8-GPU box hosts 4 of them), plus a serial run per minibatch for the speed-up
column. Prints and writes one CSV row per cell (sweep.grid_csv format plus
the minibatch) and the per-epoch metrics CSVs next to it.

Frames/s here is the reference's wall-clock training throughput of all
virtual replicas on ONE GPU (they share it), not a per-GPU bench number.
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_1507_01239_b200 import parnn as P  # noqa: E402
from paper_1507_01239_b200 import sweep as S  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workers", type=int, default=32)
    ap.add_argument("--avg-frequencies", default="1,2,4,8,16,32,64")
    ap.add_argument("--minibatches", default="256,512,1024,2048,4096")
    ap.add_argument("--per-class", type=int, default=128)
    ap.add_argument("--epochs", type=int, default=1)
    ap.add_argument("--lr-init", type=float, default=0.32)
    ap.add_argument("--separation", type=float, default=8.0)
    ap.add_argument("--optimizer", choices=["ngsgd_lowrank", "ngsgd", "sgd"], default="ngsgd_lowrank")
    ap.add_argument("--precision", choices=["bf16", "tf32", "fp32"], default="bf16")
    ap.add_argument("--dims", default="440,2048,2048,2048,2048,2048,2048,8806")
    ap.add_argument("--no-serial", action="store_true")
    ap.add_argument("--out", default="gpurun_out/cfg5_sweep")
    args = ap.parse_args()

    dims = tuple(int(x) for x in args.dims.split(","))
    ks = [int(x) for x in args.avg_frequencies.split(",")]
    bs = [int(x) for x in args.minibatches.split(",")]
    os.makedirs(args.out, exist_ok=True)
    ctx = P.Context(0)
    opts = P.TrainOptions(optimizer=P.OptimizerKind[args.optimizer], lr_schedule=P.LrVariant.exponential,
                          lr_init=args.lr_init, epochs=args.epochs, precision=P.Precision[args.precision])
    t0 = time.perf_counter()
    base = S.RunConfig(dims=dims, per_class=args.per_class, separation=args.separation, plan=P.ParallelPlan(args.workers, 4, 1024, 0),
                       opts=opts)
    S._data(base)  # generate once (shared by every cell)
    gen_s = time.perf_counter() - t0

    def runner(cfg):
        res = S.run(cfg, ctx)
        tag = f"m{cfg.plan.workers}_b{cfg.plan.minibatch}_k{cfg.plan.avg_frequency}"
        S.write_metrics_csv(res.metrics, os.path.join(args.out, f"metrics_{tag}.csv"))
        return res

    lines = []
    header = None
    for b in bs:
        cfg_b = base.with_value("minibatch", b)
        rows = S.compare_grid(cfg_b, "avg_frequency", ks, serial_baseline=not args.no_serial, runner=runner)
        text = S.grid_csv("avg_frequency", rows).splitlines()
        header = "minibatch," + text[0]
        for t in text[1:]:
            lines.append(f"{b},{t}")
            print(f"{b},{t}", flush=True)
    with open(os.path.join(args.out, "grid.csv"), "w") as f:
        f.write("\n".join([header] + lines) + "\n")
    info = {"workers": args.workers, "dims": dims, "per_class": args.per_class, "epochs": args.epochs,
            "optimizer": args.optimizer, "precision": args.precision, "lr_init": args.lr_init,
            "separation": args.separation, "avg_frequencies": ks, "minibatches": bs,
            "data_gen_seconds": gen_s, "total_seconds": time.perf_counter() - t0,
            "note": "all workers are virtual replicas on one B200; frames_per_s = frames / training wall time"}
    with open(os.path.join(args.out, "info.json"), "w") as f:
        json.dump(info, f, indent=1)
    print(json.dumps(info))


if __name__ == "__main__":
    main()
