#!/usr/bin/env python
"""Benchmark of the model-averaging DNN trainer path (BASELINE.json).

Workload (N=1): config 2 of BASELINE.json — Switchboard-shaped DNN
440-2048x6-8806 sigmoid, NG-SGD, minibatch 1024, synthetic frames from the
reference's own generate_synthetic recipe. NG-SGD is the north star's online
low-rank preconditioner by default (--optimizer ngsgd_lowrank); the
reference's kron-full NG-SGD is timed on the same data in the same run
("ngsgd_kron_full") and is selectable with --optimizer ngsgd. N>1 (torchrun): config 3 — one replica per GPU,
model averaging every 4 minibatches over NCCL (weak scaling: each GPU does
the same per-step work).

One "step" = one minibatch update on every replica (gather -> forward ->
softmax-CE -> backward -> NG precondition (+ subspace update) -> SGD), plus the
averaging event every --avg-frequency steps.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Rank 0 prints ONE JSON line (metric/value/unit/... + roofline, cpu_baseline,
e2e, clocks, gpu_launches).
"""
import argparse
import json
import os
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

DIMS = [440] + [2048] * 6 + [8806]
OPT_DESC = {"ngsgd_lowrank": "NG-SGD (online low-rank Fisher, rank 20/80, update every 4)",
            "ngsgd": "NG-SGD (the reference's kron-full Fisher)", "sgd": "plain SGD"}
METRIC = "training frames/sec (440-2048x6-8806 NG-SGD, minibatch 1024)"
UNIT = "frames/s"


def flops_per_frame(dims):
    # model GEMM flops/frame: 6*sum(din*dout) - 2*d0*d1 (layer 0 has no dA)
    return 6 * sum(dims[l] * dims[l + 1] for l in range(len(dims) - 1)) - 2 * dims[0] * dims[1]


def peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))), "measured"
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}, "fallback"


# ------------------------------------------------------------ CPU reference
def reference_sample(steps, threads=1):
    """Time the UNMODIFIED reference (oracle/_ref) on a bounded sample of the
    config-2 step: the same network with every layer width scaled by 1/8
    (55-256x6-1101), batch 1024. Per-phase times are extrapolated exactly by
    the cost model of the reference loops: forward/backward/ng_update/sgd are
    degree-2 in the widths (x64), ng_precondition (Cholesky + triangular
    solves) is degree-3 (x512)."""
    from oracle.ref_lib import RefLib, available
    if not available():
        raise RuntimeError("oracle/_ref/libparnn_ref.so missing (make -C oracle)")
    R = RefLib()
    s = 8
    dims = [max(1, d // s) for d in DIMS]
    rng = np.random.default_rng(0)
    n = 4096
    x = rng.standard_normal((n, dims[0]))
    y = rng.integers(0, dims[-1], n).astype(np.int32)
    p0 = R.init_random(dims, 1)
    t0 = time.perf_counter()
    fps_s, ph = R.time_steps(dims, p0, x, y, 1024, steps, True, threads)
    wall = time.perf_counter() - t0
    per_step = ph / steps
    est = (per_step[0] + per_step[1] + per_step[2] + per_step[4]) * s ** 2 + per_step[3] * s ** 3
    return {
        "value": 1024.0 * threads / est,
        "unit": UNIT,
        "cores": threads,
        "kind": "reference",
        "sample": (f"{steps} reference step(s) of 55-256x6-1101 NG-SGD at minibatch 1024 "
                   f"({wall:.1f} s CPU); fwd/bwd/ng_update/sgd x64 and ng_precondition x512 "
                   f"(width^2 / width^3 cost of the reference loops) -> {est:.1f} s per config-2 step"),
        "phase_seconds_extrapolated": {"forward+ce": per_step[0] * 64, "backward": per_step[1] * 64,
                                       "ng_update_state": per_step[2] * 64, "ng_precondition": per_step[3] * 512,
                                       "sgd": per_step[4] * 64},
    }


# -------------------------------------------------------------- clocks
class ClockSampler:
    def __init__(self, path):
        self.path = path
        self.proc = None

    def __enter__(self):
        q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.f = open(self.path, "w")
            self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={q}", "--format=csv,noheader,nounits",
                                          "-lms", "100"], stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            self.proc.wait()
            self.f.close()

    def summary(self, device=0):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in open(self.path):
            f = [v.strip() for v in line.split(",")]
            if len(f) < 9 or f[0] != str(device):
                continue
            try:
                sm.append(float(f[1]))
                mx = float(f[2])
            except ValueError:
                continue
            for nm, v in zip(names, f[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


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

    # synthetic Switchboard-shaped frames (generate_synthetic + split + standardize, data.cpp:124-242)
    t0 = time.perf_counter()
    train, _ = P.make_data(DIMS[-1], DIMS[0], args.per_class, 8.0, 1, 0.10, 2, True)
    shards = P.partition_rows(train.size(), world, 0)
    ds = P.DeviceDataset(ctx, train)
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
    lrs = np.full(need, 1e-3, np.float32)
    rep.upload_epoch(rows, lrs)
    rep.step(W)
    rep.sync()
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    clk = ClockSampler(os.path.join(ROOT, "gpurun_out" if os.path.isdir(os.path.join(ROOT, "gpurun_out")) else ".",
                                    f"clocks_rank{rank}.csv"))
    with clk:
        ms = P.run_steps([rep], K, args.avg_frequency, comm=comm, m_total=world)
    rep.sync()
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
        t = torch.tensor([ms], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    ms_per_step = ms / K
    value = world * B * K / (ms / 1e3)
    ce = rep.ce(W + K)
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
    peak_t = pk.get("bf16_tflops_sustained", pk["bf16_tflops"])
    achieved = (d_fl / d_n) / (d_ms / d_n / 1e3) / 1e12 if d_fl > 0 else None
    # DRAM bytes per launch of the dominant kernel from the committed ncu --set full
    # capture (dram__bytes_read.sum + dram__bytes_write.sum, profiles/)
    # algorithmic bytes of one dW launch (avg over layers): fp32 W read + write, bf16 shadow
    # write, and the two bf16 operands (B x dout, B x (din + 1))
    dw_bytes = sum(10.0 * o * (i + 1) + 2.0 * B * (o + i + 1) for i, o in zip(DIMS[:-1], DIMS[1:])) / (len(DIMS) - 1)
    traffic, traffic_src = None, None
    tpath = os.path.join(ROOT, "profiles", "dominant_traffic.json")
    if os.path.exists(tpath):
        try:
            t = json.load(open(tpath)).get(dom) or {}
            traffic, traffic_src = t.get("bytes_per_launch"), t.get("source")
        except Exception:
            traffic = None
    roofline = {"bound": "tensor", "kernel": dom, "achieved": achieved, "peak": peak_t, "unit": "TFLOP/s",
                "frac": (achieved / peak_t) if achieved else None, "traffic": traffic,
                "traffic_unit": "bytes per launch", "traffic_source": traffic_src,
                "algorithmic_bytes_per_launch": dw_bytes,
                "peak_source": f"{how} bf16_tflops_sustained (MEASURED_PEAKS.json)",
                "launches_per_step": d_n, "ms_per_step": d_ms,
                "note": ("tcgen05 GEMM region, algorithmic flops (2MNK per launch) / CUDA-event time of the region "
                         "in an eager serial profile of %d steps (one low-rank update period)" % args.profile_steps)}
    model_gemm = {"achieved": g_fl / (g_ms / 1e3) / 1e12, "peak": peak_t, "unit": "TFLOP/s",
                  "frac": g_fl / (g_ms / 1e3) / 1e12 / peak_t, "ms_per_step": g_ms,
                  "flops_per_step": g_fl, "kinds": gemm_kinds}

    # ---- end-to-end through the C ABI with host buffers: per step, host batch
    # assembly into pinned staging (double buffered), H2D (parnn_dataset_write_f32),
    # the step, and the D2H read of a step's loss (parnn_replica_step_ce). The loss
    # of step i is read after step i+1 has been queued, so the copies and the host
    # work overlap the GPU instead of serialising with it.
    e2e = None
    if not args.no_e2e:
        E = args.e2e_steps
        pins = [torch.empty((B, DIMS[0]), dtype=torch.float32, pin_memory=True) for _ in range(2)]
        pinys = [torch.empty((B,), dtype=torch.int32, pin_memory=True) for _ in range(2)]
        stage = P.DeviceDataset(ctx, P.Dataset(train.features[:2 * B], train.labels[:2 * B], DIMS[-1]))
        rep_e = P.Replica(ctx, DIMS, precision=prec, optimizer=opt, minibatch=B, max_steps=E + 4)
        rep_e.set_params(m0.params)
        rep_e.bind(stage)
        rep_e.upload_epoch(np.concatenate([np.arange(B) + (i % 2) * B for i in range(E + 4)]),
                           np.full(E + 4, 1e-3, np.float32))
        src = torch.from_numpy(np.random.default_rng(3).integers(0, train.size(), (E + 4, B)))
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

        stage_step(0)
        stage_step(1)
        rep_e.step_ce(1)  # warm (includes the low-rank init step)
        t0 = time.perf_counter()
        for i in range(2, 2 + E):
            stage_step(i)
            ce_e = rep_e.step_ce(i - 1)  # D2H of the previous step's loss
        ce_e = rep_e.step_ce(1 + E)
        e2e_s = time.perf_counter() - t0
        e2e = {"value": B * E / e2e_s, "unit": UNIT, "h2d_bytes_per_step": B * DIMS[0] * 4 + B * 4,
               "d2h_bytes_per_step": 8, "steps": E,
               "path": "host batch assembly (fp32 host frames, threaded row gather) -> pinned staging -> parnn_dataset_write_f32 (H2D) + parnn_replica_step "
                       "+ parnn_replica_step_ce (D2H loss, one step behind), wall clock",
               "last_ce": float(ce_e)}
        rep_e.close()

    cpu = None
    if world == 1 and not args.no_cpu:
        try:
            cpu = reference_sample(1)
        except Exception as e:  # reported, not fatal
            cpu = {"value": None, "unit": UNIT, "cores": 1, "kind": "reference", "sample": f"unavailable: {e}"}

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
        kron = {"optimizer": "ngsgd (kron-full, the reference's NG-SGD)", "value": B / (kms / 1e3), "unit": UNIT,
                "ms_per_step": kms, "kernels_per_step": rk.kernels_per_step(), "steps": 4,
                "timing": "CUDA events on the replica stream, graph launches"}
        rk.close()

    kps = rep.kernels_per_step()
    out.update({
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": K, "warmup": W,
        "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": args.precision, "data": f"synthetic (generate_synthetic 8806x{args.per_class}, 440-dim, s=8)",
        "config": {"workload": f"config 2: 440-2048x6-8806 sigmoid {OPT_DESC[args.optimizer]}, "
                               f"minibatch {B}, {'1 replica' if world == 1 else f'{world} replicas, averaging every {args.avg_frequency}'}",
                   "global_batch": B * world, "parallelism": f"dp{world} model-averaging",
                   "precision": f"{args.precision} operands, fp32 accumulate, fp32 NG solves",
                   "l2": "inputs larger than L2 (dataset %.0f MB + 160 MB fp32 params + NG factors per step)"
                         % (train.size() * 440 * (2 if prec == P.Precision.bf16 else 4) / 1e6),
                   "data_gen_seconds": gen_s},
        "clocks": clk.summary(local_rank),
        "gpu_launches": int(kps * K + (K // args.avg_frequency) * (0 if world == 1 else 2)),
        "kernels_per_step": kps,
        "roofline": roofline,
        "model_gemm_roofline": model_gemm,
        "model_flops_per_frame": flops_per_frame(DIMS),
        "e2e": e2e,
        "cpu_baseline": cpu,
        "ngsgd_kron_full": kron,
        "final_ce": float(ce[-1]),
        "regions_ms": {k: round(v[0], 4) for k, v in sorted(by_kind.items(), key=lambda kv: -kv[1][0])},
    })
    return out


def run_reference(args, rank, world):
    if rank != 0:
        return None
    t0 = time.perf_counter()
    samples = []
    try:
        for _ in range(args.warmup_ref):
            reference_sample(1)
        for _ in range(args.steps_ref):
            samples.append(reference_sample(1))
    except Exception as e:
        return {"impl": "reference", "unavailable": str(e).splitlines()[0]}
    v = float(np.mean([s["value"] for s in samples]))
    cpu = dict(samples[-1])
    cpu["value"] = v
    return {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": world, "steps": len(samples),
            "warmup": args.warmup_ref, "ms_per_step": 1024.0 / v * 1e3, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": "config 2: 440-2048x6-8806 sigmoid ngsgd (kron-full NG), minibatch 1024, "
                                   "reference CPU trainer (1 worker = 1 thread)", "global_batch": 1024,
                       "parallelism": "1 worker"},
            "cpu_baseline": cpu,
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "wall_seconds": time.perf_counter() - t0}


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
    ap.add_argument("--per-class", type=int, default=24)
    ap.add_argument("--profile-steps", type=int, default=4)
    ap.add_argument("--e2e-steps", type=int, default=600)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    args = ap.parse_args()
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local_rank = int(os.environ.get("LOCAL_RANK", 0))
    if args.impl == "reference":
        args.warmup_ref = 0
        args.steps_ref = max(1, min(args.steps, 3))
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
