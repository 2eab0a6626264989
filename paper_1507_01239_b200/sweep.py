"""Experiment driver around ``train_parallel``: metrics CSV, speed-up and
averaging-frequency / minibatch grids.

The reference library ships no driver; its spec describes one
(``/root/reference/SPEC.md:526-550``): ``run`` writes one ``MetricsRecord``
per epoch as CSV with the fixed header below, ``compute_speedup`` divides the
serial by the parallel wall time, and ``compare_grid`` runs one config per
value of an axis (optionally over seeds) and tabulates final CV accuracy and
speed-up with mean and standard deviation. Wall time covers the training loop
only (the reference's ``wall_seconds``, ``parallel.cpp:236-247``).

Everything here is host bookkeeping; the runs go through
``parnn.train_parallel`` / ``serial_train`` on the GPU.
"""
from __future__ import annotations

import csv
import io
import math
from dataclasses import dataclass, field, replace

from . import parnn as P

CSV_HEADER = ("epoch", "lr", "train_ce", "cv_accuracy", "wall_seconds", "workers", "avg_events")


def write_metrics_csv(metrics, path_or_buf=None) -> str:
    """One row per ``EpochMetrics`` under the fixed header.
    Floats are written with ``repr`` so the file parses back exactly."""
    buf = io.StringIO()
    w = csv.writer(buf, lineterminator="\n")
    w.writerow(CSV_HEADER)
    for m in metrics:
        w.writerow([m.epoch, repr(float(m.lr)), repr(float(m.train_ce)), repr(float(m.cv_accuracy)),
                    repr(float(m.wall_seconds)), m.workers, m.avg_events])
    text = buf.getvalue()
    if path_or_buf is not None:
        if hasattr(path_or_buf, "write"):
            path_or_buf.write(text)
        else:
            with open(path_or_buf, "w") as f:
                f.write(text)
    return text


def read_metrics_csv(text: str) -> list:
    """Inverse of ``write_metrics_csv``; a wrong header is an error naming it."""
    rows = list(csv.reader(io.StringIO(text)))
    if not rows or tuple(rows[0]) != CSV_HEADER:
        raise P.ParnnError(f"read_metrics_csv: unexpected header {rows[0] if rows else '<empty>'}")
    out = []
    for r in rows[1:]:
        if not r:
            continue
        out.append(P.EpochMetrics(int(r[0]), float(r[1]), float(r[2]), float(r[3]), float(r[4]), int(r[5]),
                                  int(r[6])))
    return out


def compute_speedup(serial_metrics, parallel_metrics):
    """(speedup, scaling) = (serial wall / parallel wall, speedup / workers)
    (SPEC.md:533-541). ``workers`` is the parallel run's worker count."""
    ts = sum(m.wall_seconds for m in serial_metrics)
    tp = sum(m.wall_seconds for m in parallel_metrics)
    if not parallel_metrics or tp <= 0.0:
        raise P.ParnnError("compute_speedup: parallel run has zero wall time")
    workers = parallel_metrics[-1].workers
    if workers < 1:
        raise P.ParnnError(f"compute_speedup: invalid worker count {workers}")
    speedup = ts / tp
    return speedup, speedup / workers


@dataclass
class RunConfig:
    """One training run: data recipe, network, plan and options."""
    dims: tuple = (440, 512, 512, 1000)
    per_class: int = 100
    separation: float = 8.0
    data_seed: int = 1
    cv_fraction: float = 0.10
    split_seed: int = 2
    init_seed: int = 7
    plan: P.ParallelPlan = field(default_factory=lambda: P.ParallelPlan(1, 4, 256, 0))
    opts: P.TrainOptions = field(default_factory=lambda: P.TrainOptions(epochs=1))

    def with_value(self, axis: str, value) -> "RunConfig":
        """Set ``axis`` on the config, the plan or the options (first match)."""
        if axis in RunConfig.__dataclass_fields__ and axis not in ("plan", "opts"):
            return replace(self, **{axis: value})
        if axis in P.ParallelPlan.__dataclass_fields__:
            return replace(self, plan=replace(self.plan, **{axis: value}))
        if axis in P.TrainOptions.__dataclass_fields__:
            return replace(self, opts=replace(self.opts, **{axis: value}))
        raise P.ParnnError(f"compare_grid: unknown axis '{axis}'")


_data_cache: dict = {}
_device_cache: dict = {}


def _key(cfg: RunConfig):
    return (cfg.dims[-1], cfg.dims[0], cfg.per_class, cfg.separation, cfg.data_seed, cfg.cv_fraction, cfg.split_seed)


def _data(cfg: RunConfig):
    key = _key(cfg)
    if key not in _data_cache:
        _data_cache.clear()
        _device_cache.clear()
        _data_cache[key] = P.make_data(*key, True)
    return _data_cache[key]


def _device_data(cfg: RunConfig, ctx: P.Context):
    """The run's train / CV sets uploaded once per (data recipe, context)."""
    train, cv = _data(cfg)
    key = (_key(cfg), id(ctx))
    if key not in _device_cache:
        _device_cache.clear()
        _device_cache[key] = (ctx, P.DeviceDataset(ctx, train), P.DeviceDataset(ctx, cv) if cv.size() else None)
    return _device_cache[key][1:]


_models: dict = {}


def run(cfg: RunConfig, ctx: P.Context | None = None) -> P.TrainResult:
    """SPEC.md:526-532 ``run`` minus file plumbing: ``train_parallel`` of
    the config from ``init_random(dims, init_seed)``. With a context the data
    set stays resident across runs."""
    train, cv = _data(cfg)
    mkey = (tuple(cfg.dims), cfg.init_seed)
    if mkey not in _models:
        _models.clear()
        _models[mkey] = P.init_random(list(cfg.dims), seed=cfg.init_seed)
    dd = _device_data(cfg, ctx) if ctx is not None else None
    return P.train_parallel(cfg.plan, _models[mkey], train, cv, cfg.opts, ctx=ctx, device_data=dd)


@dataclass
class GridRow:
    value: object
    seeds: int
    final_ce: float
    final_ce_std: float
    cv_accuracy: float
    cv_accuracy_std: float
    frames_per_s: float
    speedup: float
    wall_seconds: float
    error: str = ""


def _mean_std(xs):
    if not xs:
        return math.nan, math.nan
    mu = sum(xs) / len(xs)
    return mu, (math.sqrt(sum((x - mu) ** 2 for x in xs) / (len(xs) - 1)) if len(xs) > 1 else 0.0)


def compare_grid(base: RunConfig, axis: str, values, seeds=(0,), serial_baseline: bool = True,
                 runner=run) -> list:
    """one run per (value, seed); per value the mean ± std of
    the final train CE and CV accuracy, frames/s and the speed-up against a
    serial run of the same config (one worker). A failing cell becomes a row
    carrying its error text (partial table)."""
    rows = []
    serial_cache = {}
    for v in values:
        ces, accs, fps, sps, walls, err = [], [], [], [], [], ""
        for s in seeds:
            cfg = base.with_value(axis, v)
            cfg = replace(cfg, plan=replace(cfg.plan, base_seed=s))
            try:
                res = runner(cfg)
                ms = res.metrics
                wall = sum(m.wall_seconds for m in ms)
                train, _ = _data(cfg)
                per_worker = (train.size() // cfg.plan.workers) // cfg.plan.minibatch * cfg.plan.minibatch
                frames = per_worker * cfg.plan.workers * len(ms)
                ces.append(ms[-1].train_ce)
                accs.append(ms[-1].cv_accuracy)
                fps.append(frames / wall if wall > 0 else math.nan)
                walls.append(wall)
                if serial_baseline:
                    skey = (repr(replace(cfg.plan, workers=1, avg_frequency=1)), repr(cfg.opts), cfg.dims)
                    if skey not in serial_cache:
                        scfg = replace(cfg, plan=replace(cfg.plan, workers=1, avg_frequency=1))
                        serial_cache[skey] = runner(scfg).metrics
                    sps.append(compute_speedup(serial_cache[skey], ms)[0])
            except P.ParnnError as e:  # partial table with a failure marker
                err = str(e)
        ce, ce_sd = _mean_std(ces)
        acc, acc_sd = _mean_std(accs)
        rows.append(GridRow(v, len(ces), ce, ce_sd, acc, acc_sd, _mean_std(fps)[0],
                            _mean_std(sps)[0] if sps else math.nan, _mean_std(walls)[0], err))
    return rows


def grid_csv(axis: str, rows) -> str:
    buf = io.StringIO()
    w = csv.writer(buf, lineterminator="\n")
    w.writerow([axis, "seeds", "final_train_ce", "final_train_ce_std", "cv_accuracy", "cv_accuracy_std",
                "frames_per_s", "speedup", "wall_seconds", "error"])
    for r in rows:
        w.writerow([r.value, r.seeds, r.final_ce, r.final_ce_std, r.cv_accuracy, r.cv_accuracy_std,
                    r.frames_per_s, r.speedup, r.wall_seconds, r.error])
    return buf.getvalue()
