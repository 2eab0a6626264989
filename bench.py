#!/usr/bin/env python
"""Benchmark of the model-averaging DNN trainer path (BASELINE.json).

Workload: config 2 of BASELINE.json at N=1 -- Switchboard-shaped DNN
440-2048x6-8806 sigmoid, NG-SGD, minibatch 1024 -- and config 3 at N>1 (one
replica per GPU, model averaging every 4 minibatches over NCCL; weak scaling:
every GPU does the same per-step work). Synthetic frames come from the
reference's own generate_synthetic + split_cv + standardize recipe.

NG-SGD is the north star's online low-rank preconditioner (--optimizer
ngsgd_lowrank, the default); the reference's own kron-full NG-SGD runs on the
same data in the same process ("ngsgd_kron_full") and is selectable with
--optimizer ngsgd.

One "step" = one minibatch update on every replica (gather -> forward ->
softmax-CE -> backward -> NG precondition (+ subspace update) -> SGD), plus
the averaging event every --avg-frequency steps.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

With --gpus N > 1 and no torchrun environment, the script relaunches itself
under torch.distributed.run with N ranks (127.0.0.1). Rank 0 prints ONE JSON
line (metric/value/unit/... + roofline, cpu_baseline, e2e, clocks,
gpu_launches).

--impl reference times the UNMODIFIED reference (oracle/_ref, compiled from
its sources): one true-width config-2 minibatch with its own kron-full NG-SGD
on all host cores. One such step takes minutes of CPU time, so the reference
line reports steps = 1, warmup = 0 (nothing is extrapolated).
"""
import argparse
import json
import math
import os
import socket
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

DIMS = [440] + [2048] * 6 + [8806]
OPT_DESC = {"ngsgd_lowrank": "ngsgd_lowrank: online low-rank Fisher NG-SGD (north star; rank 20/80, subspace "
                             "update every 4 steps)",
            "ngsgd": "ngsgd: the reference's kron-full Kronecker-factored NG-SGD (optimizer.cpp:44-157)",
            "sgd": "sgd: plain SGD"}
METRIC = "training frames/sec (440-2048x6-8806 NG-SGD, minibatch 1024)"
UNIT = "frames/s"
# Calibrated with scripts/calibrate_cfg2.py (SURVEY §8d "Calibrate s"; profiles/
# r2_calibration.txt): at s = 20 and 128 frames per class the low-rank NG-SGD (lr 10,
# exponential schedule over 6 epochs) takes the frame CE from ln 8806 = 9.08 to ~0.3
# while plain SGD stays at ln 8806; s <= 16 learns only late, s >= 32 is separable
# within 2 epochs; lr >= 20 diverges.
SEPARATION = 20.0
LR_INIT = 10.0


def flops_per_frame(dims):
    # model GEMM flops/frame: 6*sum(din*dout) - 2*d0*d1 (layer 0 has no dA)
    return 6 * sum(dims[l] * dims[l + 1] for l in range(len(dims) - 1)) - 2 * dims[0] * dims[1]


def peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))), "measured (MEASURED_PEAKS.json)"
    except Exception:
        return ({"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0},
                "fallback (B200_PROFILING.md)")


def workload_config(args, world):
    """The workload both arms run (identical dict in both JSON lines)."""
    n = DIMS[-1] * args.per_class
    n_train = n - math.ceil(0.10 * n)  # split_cv takes ceil(f N) to CV (data.cpp:178-179)
    reps = "1 replica" if world == 1 else f"{world} replicas (one per GPU), averaging every {args.avg_frequency}"
    return {
        "workload": f"config {2 if world == 1 else 3}: 440-2048x6-8806 sigmoid NG-SGD, minibatch "
                    f"{args.minibatch}, {reps}",
        "global_batch": args.minibatch * world,
        "parallelism": f"dp{world} model-averaging",
        "avg_frequency": args.avg_frequency,
        "data": (f"generate_synthetic({DIMS[-1]} classes x {args.per_class}, {DIMS[0]}-dim, s={SEPARATION:g}, "
                 f"seed 1) -> split_cv(0.1, seed 2) -> standardize (on the device): {n_train} train frames"),
        "l2": "inputs larger than L2: the resident training set is %.0f MB (bf16) and each step streams 160 MB of "
              "fp32 parameters" % (n_train * 440 * 2 / 1e6),
    }


# ------------------------------------------------------------ CPU reference
def reference_step(per_class, threads=None):
    """One TRUE-WIDTH config-2 minibatch of the UNMODIFIED reference
    (oracle/_ref): worker_epoch's body (parallel.cpp:117-130) with the
    reference's own kron-full NG-SGD, at 440-2048x6-8806, batch 1024, on the
    same synthetic frames as our arm, built from the reference's public
    functions and spread over all host cores (ref_time_step_threaded; equal to
    the single-threaded reference step up to fp64 summation order). Nothing is
    extrapolated: the value is 1024 frames / the measured wall time."""
    from oracle.ref_lib import RefLib, available
    if not available():
        raise RuntimeError("oracle/_ref/libparnn_ref.so missing (make -C oracle)")
    from paper_1507_01239_b200 import parnn as P
    R = RefLib()
    threads = threads or os.cpu_count() or 1
    train, _ = P.make_data(DIMS[-1], DIMS[0], per_class, SEPARATION, 1, 0.10, 2, True)
    order = P.minibatch_rows(train.size(), 1024, int(P.rng_u64(0, 1)[0]))[0].astype(np.int64)
    x, y = train.features[order], train.labels[order]
    p0 = R.init_random(DIMS, 7)
    wall, ph, _, ce = R.time_step_threaded(DIMS, p0, x, y, True, threads)
    names = ["forward+ce", "backward", "ng_moments", "ng_factor+solve1+bias", "ng_solve2", "ng_gamma", "sgd"]
    return {
        "value": 1024.0 / wall, "unit": UNIT, "cores": threads, "kind": "reference",
        "sample": ("one full config-2 minibatch (440-2048x6-8806, batch 1024, kron-full NG-SGD, fp64) of the "
                   "unmodified reference's own functions on %d host threads: %.1f s wall, no extrapolation"
                   % (threads, wall)),
        "phase_seconds": {n: round(float(t), 3) for n, t in zip(names, ph)},
        "batch_ce": ce, "wall_seconds": wall,
    }


# -------------------------------------------------------------- clocks
class ClockSampler:
    """NVML polling thread (~1 ms) over the timed region: SM clock, max clock
    and the throttle reasons seen while the GPU is busy."""
    BITS = {0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown", 0x20: "sw_thermal_slowdown", 0x4: "sw_power_cap",
            0x80: "hw_power_brake_slowdown"}

    def __init__(self, device):
        self.device, self.samples, self.reasons, self.max_mhz = device, [], set(), None
        self.err = None

    def __enter__(self):
        self.stop = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.device)
            self.max_mhz = float(pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM))

            def poll():
                while not self.stop.is_set():
                    try:
                        util = pynvml.nvmlDeviceGetUtilizationRates(h).gpu
                        mhz = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
                        rs = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
                    except Exception as e:  # noqa: BLE001
                        self.err = str(e)
                        return
                    self.samples.append((float(mhz), int(util)))
                    for bit, name in self.BITS.items():
                        if rs & bit:
                            self.reasons.add(name)
                    time.sleep(0.001)

            self.th = threading.Thread(target=poll, daemon=True)
            self.th.start()
        except Exception as e:  # noqa: BLE001
            self.err, self.th = str(e), None
        return self

    def __exit__(self, *a):
        self.stop.set()
        if getattr(self, "th", None):
            self.th.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons), "samples": 0,
                    "note": self.err or "no samples"}
        busy = [m for m, u in self.samples if u > 0] or [m for m, _ in self.samples]
        return {"sm_mhz": float(np.median(busy)), "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(self.samples), "samples_busy": len(busy), "source": "NVML, ~1 ms polling"}


# -------------------------------------------------------------- our arm
def run_ours(args, rank, world, local_rank):
    import torch
    from paper_1507_01239_b200 import parnn as P

    torch.cuda.set_device(local_rank)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    prec = P.Precision.bf16 if args.precision == "bf16" else P.Precision.tf32
    opt = P.OptimizerKind[args.optimizer]
    B, K, W = args.minibatch, args.steps, args.warmup
    ctx = P.Context(local_rank)
    comm = None
    if world > 1:
        uid = [P.Comm.unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        comm = P.Comm(ctx, uid[0], world, rank)

    def max_over_ranks(v):
        if not dist:
            return v
        t = torch.tensor([v], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    # synthetic Switchboard-shaped frames (generate_synthetic + split + standardize, data.cpp:124-242,
    # generated on the device); worker r trains on shard r of partition_data (parallel.cpp:61-77)
    t0 = time.perf_counter()
    ds, cv_ds = P.DeviceDataset.generate(ctx, DIMS[-1], DIMS[0], args.per_class, SEPARATION, 1, 0.10, 2, True)
    shards = P.partition_rows(ds.n, world, 0)
    gen_s = time.perf_counter() - t0
    m0 = P.init_random(DIMS, seed=7)
    rep = P.Replica(ctx, DIMS, precision=prec, optimizer=opt, minibatch=B, max_steps=W + K + 8)
    rep.set_params(m0.params)
    rep.bind(ds)
    S = shards.shape[1]
    order = P.minibatch_rows(S, B, int(P.rng_u64(rank, 1)[0]))
    need = W + K + 8
    rows = shards[rank][order.ravel().astype(np.int64)]
    rows = np.resize(rows, need * B)
    lrs = np.full(need, LR_INIT * 0.01 ** 0.5, np.float32)  # the exponential schedule's mid-run rate
    rep.upload_epoch(rows, lrs)
    if W:
        P.run_steps([rep], W, args.avg_frequency, comm=comm, m_total=world)  # warm-up, averaging included
    rep.sync()
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local_rank) as clk:
        ms = P.run_steps([rep], K, args.avg_frequency, comm=comm, m_total=world)  # CUDA events, this rank
    rep.sync()
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    ms = max_over_ranks(ms)
    ms_per_step = ms / K
    value = world * B * K / (ms / 1e3)
    ce = rep.ce(W + K)

    # ---- averaging alone: NVLink bus bandwidth (N > 1)
    avg = None
    if world > 1:
        a_ms, a_bytes = P.time_average([rep], comm=comm, m_total=world, iters=10)
        a_ms = max_over_ranks(a_ms)
        avg = {"ms_per_event": a_ms, "bytes_per_event": a_bytes, "events_per_step": 1.0 / args.avg_frequency,
               "bus_gbs": 2.0 * (world - 1) / world * a_bytes / (a_ms / 1e3) / 1e9,
               "how": "per-layer ncclAllReduce(ncclAvg) buckets + bf16 copy, 10 back-to-back events, CUDA events, "
                      "max over ranks; bus GB/s = 2(n-1)/n * bytes / time"}

    # ---- end-to-end through the C ABI with host buffers (every rank): per step, host
    # batch assembly into pinned staging (double buffered), H2D (parnn_dataset_write_f32),
    # the step, the averaging event every avg_frequency steps (parnn_averager_run), and the
    # D2H read of a step's loss (parnn_replica_step_ce, one step behind, so copies and
    # host work overlap the GPU). Wall clock, max over ranks.
    e2e = None
    if not args.no_e2e:
        E = args.e2e_steps
        pins = [torch.empty((B, DIMS[0]), dtype=torch.float32, pin_memory=True) for _ in range(2)]
        pinys = [torch.empty((B,), dtype=torch.int32, pin_memory=True) for _ in range(2)]
        train = ds.download()  # host-resident frames (fp32, as on the device)
        stage = P.DeviceDataset(ctx, P.Dataset(train.features[:2 * B], train.labels[:2 * B], DIMS[-1]))
        rep_e = P.Replica(ctx, DIMS, precision=prec, optimizer=opt, minibatch=B, max_steps=E + 4)
        rep_e.set_params(m0.params)
        rep_e.bind(stage)
        rep_e.upload_epoch(np.concatenate([np.arange(B) + (i % 2) * B for i in range(E + 4)]),
                           np.full(E + 4, LR_INIT * 0.01 ** 0.5, np.float32))
        avg_e = P.Averager([rep_e], comm=comm, m_total=world)
        src = torch.from_numpy(shards[rank][np.random.default_rng(3 + rank).integers(0, S, (E + 4, B))].astype(np.int64))
        # host-resident training frames in the device dataset's element type (fp32),
        # converted once like the upload in parnn_dataset_create; the per-step row
        # gather runs on the host's threads straight into the pinned staging buffer
        host_x = torch.from_numpy(np.ascontiguousarray(train.features, dtype=np.float32))
        host_y = torch.from_numpy(np.ascontiguousarray(train.labels, dtype=np.int32))

        def stage_step(i):
            torch.index_select(host_x, 0, src[i], out=pins[i % 2])  # host-side batch assembly
            torch.index_select(host_y, 0, src[i], out=pinys[i % 2])
            stage.write_rows(pins[i % 2].numpy(), pinys[i % 2].numpy(), row0=(i % 2) * B)  # H2D of this step's inputs
            rep_e.step(1)
            if (i + 1) % args.avg_frequency == 0:
                avg_e.run()

        stage_step(0)
        stage_step(1)
        rep_e.step_ce(1)  # warm (includes the low-rank init step)
        if dist:
            dist.barrier()
        t0 = time.perf_counter()
        for i in range(2, 2 + E):
            stage_step(i)
            ce_e = rep_e.step_ce(i - 1)  # D2H of the previous step's loss
        ce_e = rep_e.step_ce(1 + E)
        e2e_s = max_over_ranks(time.perf_counter() - t0)
        e2e = {"value": world * B * E / e2e_s, "unit": UNIT, "h2d_bytes_per_step": B * DIMS[0] * 4 + B * 4,
               "d2h_bytes_per_step": 8, "steps": E,
               "path": "host batch assembly (fp32 host frames, threaded row gather) -> pinned staging -> "
                       "parnn_dataset_write_f32 (H2D) + parnn_replica_step (+ parnn_averager_run every "
                       f"{args.avg_frequency}) + parnn_replica_step_ce (D2H loss, one step behind); wall clock, "
                       "max over ranks",
               "last_ce": float(ce_e)}
        avg_e.close()
        rep_e.close()

    out = {"_rank": rank}
    if rank != 0:
        return out

    # ---- per-region live timing (CUDA events on the replica stream) -> roofline
    prof = rep.profile(args.profile_steps)
    by_kind = {}
    for name, t, fl in prof:
        kind = name.split(":")[0]
        a = by_kind.setdefault(kind, [0.0, 0.0, 0])
        a[0] += t
        a[1] += fl
        a[2] += 1
    pk, how = peaks()
    # dominant tensor-core kernel of the step (the roofline the path is held to);
    # the SIMT regions (NG subspace eigensolver, softmax, gather) are listed in regions_ms
    dom = max((k for k in by_kind if k.startswith("gemm_")), key=lambda k: by_kind[k][0])
    d_ms, d_fl, d_n = by_kind[dom]
    gemm_kinds = [k for k in by_kind if k.startswith("gemm_") and k != "gemm_ng_moments"]
    g_ms = sum(by_kind[k][0] for k in gemm_kinds)
    g_fl = sum(by_kind[k][1] for k in gemm_kinds)
    burst = pk["bf16_tflops"]
    sustained = pk.get("bf16_tflops_sustained", burst)
    achieved = (d_fl / d_n) / (d_ms / d_n / 1e3) / 1e12 if d_fl > 0 else None
    # algorithmic bytes per launch of the dominant kind (avg over layers)
    pairs = list(zip(DIMS[:-1], DIMS[1:]))
    alg_bytes = {
        # dW + SGD: fp32 W read + write, bf16 shadow write, the two bf16 operands (B x dout, B x (din + 1))
        "gemm_dw_sgd": sum(10.0 * o * (i + 1) + 2.0 * B * (o + i + 1) for i, o in pairs) / len(pairs),
        # forward: bf16 X (B x din) and W (dout x din) read, bf16 activations (B x dout) written;
        # the output layer writes fp32 logits
        "gemm_fwd": sum(2.0 * B * i + 2.0 * o * i + (4.0 if k == len(pairs) - 1 else 2.0) * B * o
                        for k, (i, o) in enumerate(pairs)) / len(pairs),
        # dA: bf16 dZ (B x dout) and W read, bf16 dA (B x din) written
        "gemm_da": sum(2.0 * B * o + 2.0 * o * i + 2.0 * B * i for i, o in pairs[1:]) / max(1, len(pairs) - 1),
    }
    # DRAM bytes per launch of the dominant kernel from the committed ncu --set full capture
    traffic, traffic_src = None, None
    tpath = os.path.join(ROOT, "profiles", "dominant_traffic.json")
    if os.path.exists(tpath):
        try:
            t = json.load(open(tpath)).get(dom) or {}
            traffic, traffic_src = t.get("bytes_per_launch"), t.get("source")
        except Exception:
            traffic = None
    step_flops = flops_per_frame(DIMS) * B
    roofline = {"bound": "tensor", "kernel": dom, "achieved": achieved, "peak": burst, "unit": "TFLOP/s",
                "frac": (achieved / burst) if achieved else None, "traffic": traffic,
                "traffic_unit": "DRAM bytes per launch", "traffic_source": traffic_src,
                "algorithmic_bytes_per_launch": alg_bytes.get(dom),
                "peak_source": f"{how} bf16_tflops (burst: each launch is timed alone in the eager profile)",
                "launches_per_step": d_n, "ms_per_step": d_ms,
                "note": ("tcgen05 GEMM region, algorithmic flops (2MNK per launch) / CUDA-event time of the region "
                         "in an eager serial profile of %d steps (one low-rank update period)" % args.profile_steps),
                "step": {"achieved": step_flops / (ms_per_step / 1e3) / 1e12, "peak": sustained,
                         "frac": step_flops / (ms_per_step / 1e3) / 1e12 / sustained,
                         "note": "whole step: model GEMM flops per minibatch (2.376e8 x B) / the timed ms_per_step, "
                                 "against bf16_tflops_sustained (a long back-to-back run)"}}
    model_gemm = {"achieved": g_fl / (g_ms / 1e3) / 1e12, "peak": burst, "unit": "TFLOP/s",
                  "frac": g_fl / (g_ms / 1e3) / 1e12 / burst, "ms_per_step": g_ms,
                  "flops_per_step": g_fl, "kinds": gemm_kinds}

    # ---- the metric's "final frame CE": train_parallel for a fixed number of epochs on
    # the same data (train_loop semantics: per-epoch forced average, CV accuracy on
    # rank 0 outside the wall time, exponential LR), low-rank NG-SGD and plain SGD
    conv = None
    if world == 1 and args.epochs > 0:
        conv = {"epochs": args.epochs, "lr_init": LR_INIT, "schedule": "exponential", "minibatch": B,
                "avg_frequency": args.avg_frequency}
        m0c = P.init_random(DIMS, seed=7)
        for name in ("ngsgd_lowrank", "sgd"):
            o = P.TrainOptions(optimizer=P.OptimizerKind[name], lr_init=LR_INIT, epochs=args.epochs,
                               precision=prec)
            res = P.train_parallel(P.ParallelPlan(1, args.avg_frequency, B, 5), m0c, None, None, o, ctx=ctx,
                                   device_data=(ds, cv_ds))
            frames = sum((ds.n // B) * B for _ in res.metrics)
            conv[name] = {"train_ce": [round(float(m.train_ce), 4) for m in res.metrics],
                          "cv_accuracy": [round(float(m.cv_accuracy), 4) for m in res.metrics],
                          "final_ce": float(res.metrics[-1].train_ce),
                          "frames_per_s": frames / sum(m.wall_seconds for m in res.metrics)}

    cpu = None
    if world == 1 and not args.no_cpu:
        try:
            cpu = reference_step(args.per_class)
        except Exception as e:  # reported, not fatal
            cpu = {"value": None, "unit": UNIT, "cores": os.cpu_count(), "kind": "reference",
                   "sample": f"unavailable: {e}"}

    # ---- the reference's own NG variant (kron-full) on the same data, same clock
    kron = None
    if world == 1 and not args.no_kron and args.optimizer != "ngsgd":
        rk = P.Replica(ctx, DIMS, precision=prec, optimizer=P.OptimizerKind.ngsgd, minibatch=B, max_steps=8)
        rk.set_params(m0.params)
        rk.bind(ds)
        rk.upload_epoch(rows[:8 * B], lrs[:8])
        rk.step(2)
        rk.sync()
        kms = rk.time_steps(4) / 4
        kron = {"optimizer": OPT_DESC["ngsgd"], "value": B / (kms / 1e3), "unit": UNIT,
                "ms_per_step": kms, "kernels_per_step": rk.kernels_per_step(), "steps": 4,
                "timing": "CUDA events on the replica stream, graph launches",
                "vs_cpu_reference": (B / (kms / 1e3)) / cpu["value"] if cpu and cpu.get("value") else None,
                "note": "like-for-like: the same NG-SGD algorithm as the reference arm (bf16 operands here)"}
        rk.close()

    # ---- the kron-full NG in fp32 mode (3xTF32 everywhere: the mode pinned to the
    # compiled reference over whole config-1 runs, tests/test_config_parity.py)
    kron32 = None
    if world == 1 and not args.no_kron:
        rk = P.Replica(ctx, DIMS, precision=P.Precision.fp32, optimizer=P.OptimizerKind.ngsgd, minibatch=B,
                       max_steps=8)
        rk.set_params(m0.params)
        rk.bind(ds)
        rk.upload_epoch(rows[:8 * B], lrs[:8])
        rk.step(2)
        rk.sync()
        kms32 = rk.time_steps(4) / 4
        kron32 = {"optimizer": OPT_DESC["ngsgd"], "precision": "fp32 (3xTF32 operands and solves)",
                  "value": B / (kms32 / 1e3), "unit": UNIT, "ms_per_step": kms32, "steps": 4,
                  "timing": "CUDA events on the replica stream, graph launches"}
        rk.close()

    # ---- config-4 CD-1 pretraining (greedy_pretrain, pretrain.cpp:162-207) at the
    # config's layer shapes: device time of the graph-launched CD-1 epochs
    cd1 = None
    if world == 1 and not args.no_cd1:
        xs = np.random.default_rng(0).standard_normal((16384, DIMS[0]))
        cdims = [DIMS[0], 2048, 2048, 2048, 10]
        cd1 = {"workload": "greedy_pretrain 440-2048-2048-2048 (3 RBMs: 1 Gaussian-Bernoulli 440x2048, 2 Bernoulli "
                           "2048x2048) on 16384 frames x 2 epochs, batch 128",
               "flop_note": "10 v h flop per frame per RBM (SURVEY 8(d))"}
        for pn in ("bf16", "tf32"):
            pr = P.Precision[pn]
            P.greedy_pretrain(cdims[:3], xs[:2048], P.PretrainOptions(1), seed=1, precision=pr, ctx=ctx)
            P.greedy_pretrain(cdims, xs, P.PretrainOptions(2), seed=3, precision=pr, ctx=ctx)
            st = P.pretrain_last_stats()
            cd1[pn] = {"value": st["cd1_flop"] / st["cd1_device_seconds"] / 1e12, "unit": "TFLOP/s",
                       "us_per_step": st["cd1_device_seconds"] / st["cd1_steps"] * 1e6, "steps": st["cd1_steps"]}

    kps = rep.kernels_per_step()
    events = -(-K // args.avg_frequency)
    avg_kernels = 0 if world == 1 else (len(DIMS) - 1) * (2 if prec == P.Precision.bf16 else 1)
    out.update({
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": K, "warmup": W,
        "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": args.precision, "data": "synthetic",
        "optimizer": OPT_DESC[args.optimizer],
        "precision": f"{args.precision} operands, fp32 accumulate, fp32 master weights and NG solves",
        "config": workload_config(args, world),
        "clocks": clk.summary(),
        "gpu_launches": int(kps * K + events * avg_kernels),
        "kernels_per_step": kps,
        "roofline": roofline,
        "model_gemm_roofline": model_gemm,
        "model_flops_per_frame": flops_per_frame(DIMS),
        "averaging": avg,
        "e2e": e2e,
        "cpu_baseline": cpu,
        "ngsgd_kron_full": kron,
        "ngsgd_kron_full_fp32": kron32,
        "cd1_pretrain": cd1,
        "final_ce": float(ce[-1]),
        "convergence": conv,
        "data_gen_seconds": gen_s,
        "regions_ms": {k: round(v[0], 4) for k, v in sorted(by_kind.items(), key=lambda kv: -kv[1][0])},
    })
    return out


def run_reference(args, rank, world):
    """The reference arm: the unmodified reference (oracle/_ref) on this box's
    host cores, on the same workload dict as our arm. Rank 0 alone runs it.
    One true-width step; at N > 1 the host's cores are already saturated by one
    replica's step (N replicas take N times as long on the same cores), so the
    frames/s of the whole job is the same as at N = 1 and one step is timed."""
    if rank != 0:
        return None
    try:
        s = reference_step(args.per_class)
    except Exception as e:
        return {"impl": "reference", "unavailable": str(e).splitlines()[0]}
    v = s["value"]
    return {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": world, "steps": 1,
            "warmup": 0, "ms_per_step": s["wall_seconds"] * 1e3, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "optimizer": OPT_DESC["ngsgd"],
            "precision": "fp64 (the reference's only arithmetic)",
            "config": workload_config(args, world),
            "cpu_baseline": s,
            "replicas_timed": 1,
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}


def spawn(args_list, n):
    """--gpus N without a torchrun environment: relaunch under torch.distributed.run."""
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + args_list
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=600)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--precision", choices=["bf16", "tf32"], default="bf16")
    ap.add_argument("--optimizer", choices=["ngsgd_lowrank", "ngsgd", "sgd"], default="ngsgd_lowrank",
                    help="ngsgd_lowrank: the north star's online low-rank NG-SGD (default); ngsgd: the "
                         "reference's kron-full NG-SGD; sgd: plain SGD")
    ap.add_argument("--no-kron", action="store_true", help="skip the kron-full NG-SGD side measurement")
    ap.add_argument("--minibatch", type=int, default=1024)
    ap.add_argument("--avg-frequency", type=int, default=4)
    ap.add_argument("--per-class", type=int, default=128)
    ap.add_argument("--epochs", type=int, default=6, help="epochs of the final-CE run (0 = skip)")
    ap.add_argument("--profile-steps", type=int, default=4)
    ap.add_argument("--e2e-steps", type=int, default=600)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-cd1", action="store_true", help="skip the config-4 CD-1 pretraining measurement")
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(spawn(sys.argv[1:], args.gpus))
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local_rank = int(os.environ.get("LOCAL_RANK", 0))
    if args.impl == "reference":
        out = run_reference(args, rank, world)
        if out is not None:
            print(json.dumps(out), flush=True)
        return
    out = run_ours(args, rank, world, local_rank)
    if rank == 0:
        out.pop("_rank", None)
        print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
