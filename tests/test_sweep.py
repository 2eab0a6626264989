"""Experiment driver (paper_1507_01239_b200/sweep.py): the SPEC.md:526-550
examples for the metrics CSV, compute_speedup and compare_grid. CPU tests use
an injected runner; the GPU test runs a small averaging-frequency grid through
train_parallel."""
import math

import pytest

from paper_1507_01239_b200 import parnn as P
from paper_1507_01239_b200 import sweep as S


def _metrics(walls, workers=1):
    return [P.EpochMetrics(i, 0.32 * 0.5 ** i, 6.9 - 0.1 * i, 0.01 * i, w, workers, 3 * i) for i, w in enumerate(walls)]


def test_metrics_csv_round_trip_and_header():
    ms = _metrics([1.25, 0.1 + 0.2, 1e-300], workers=4)
    text = S.write_metrics_csv(ms)
    assert text.splitlines()[0] == "epoch,lr,train_ce,cv_accuracy,wall_seconds,workers,avg_events"
    assert S.read_metrics_csv(text) == ms  # exact round trip (repr floats)
    assert S.write_metrics_csv([]).strip() == ",".join(S.CSV_HEADER)  # epochs = 0: empty body
    with pytest.raises(P.ParnnError, match="unexpected header"):
        S.read_metrics_csv("a,b\n1,2\n")


def test_compute_speedup_spec_examples():
    assert S.compute_speedup(_metrics([10.0]), _metrics([10.0])) == (1.0, 1.0)  # identical runs
    sp, sc = S.compute_speedup(_metrics([60.0, 40.0]), _metrics([15.0, 10.0], workers=4))
    assert sp == pytest.approx(4.0) and sc == pytest.approx(1.0)  # serial 100 s, parallel 25 s on 4
    with pytest.raises(P.ParnnError, match="zero wall time"):
        S.compute_speedup(_metrics([1.0]), _metrics([0.0], workers=2))


def test_run_config_axes():
    base = S.RunConfig()
    assert base.with_value("avg_frequency", 16).plan.avg_frequency == 16
    assert base.with_value("optimizer", P.OptimizerKind.sgd).opts.optimizer == P.OptimizerKind.sgd
    assert base.with_value("per_class", 7).per_class == 7
    with pytest.raises(P.ParnnError, match="unknown axis 'colour'"):
        base.with_value("colour", 1)


def test_compare_grid_with_injected_runner():
    calls = []

    def runner(cfg):
        calls.append((cfg.plan.workers, cfg.plan.avg_frequency, cfg.plan.base_seed))
        if cfg.plan.avg_frequency == 99:
            raise P.ParnnError("train_parallel: boom")
        w = cfg.plan.workers
        wall = 8.0 / w if w > 1 else 8.0
        ce = 5.0 + 0.01 * cfg.plan.avg_frequency + 0.001 * cfg.plan.base_seed
        return P.TrainResult(None, [P.EpochMetrics(0, 0.32, ce, 0.5, wall, w, 1)], wall)

    base = S.RunConfig(dims=(12, 8, 10), per_class=20, plan=P.ParallelPlan(4, 1, 8, 0))
    rows = S.compare_grid(base, "avg_frequency", [1, 4, 99], seeds=(0, 1), runner=runner)
    assert [r.value for r in rows] == [1, 4, 99]
    assert rows[0].seeds == 2 and rows[0].speedup == pytest.approx(4.0)
    assert rows[1].final_ce == pytest.approx(5.04 + 0.0005) and rows[1].final_ce_std > 0
    assert rows[2].seeds == 0 and "boom" in rows[2].error and math.isnan(rows[2].final_ce)  # partial table
    # the serial baseline is run once per (plan, options): base seeds 0 and 1
    assert sum(1 for c in calls if c[0] == 1) == 2
    assert S.grid_csv("avg_frequency", rows).splitlines()[0].startswith("avg_frequency,seeds,final_train_ce")
    # single value, single seed: identical to a plain run
    one = S.compare_grid(base, "avg_frequency", [4], serial_baseline=False, runner=runner)
    assert one[0].final_ce == runner(base.with_value("avg_frequency", 4)).metrics[-1].train_ce


@pytest.mark.gpu
def test_compare_grid_on_gpu(ctx):
    base = S.RunConfig(dims=(40, 64, 64, 20), per_class=120, separation=8.0,
                       plan=P.ParallelPlan(4, 1, 32, 0),
                       opts=P.TrainOptions(optimizer=P.OptimizerKind.ngsgd_lowrank, lr_schedule=P.LrVariant.exponential,
                                           lr_init=0.32, epochs=2, precision=P.Precision.fp32, ng_rank_in=8,
                                           ng_rank_out=8))
    rows = S.compare_grid(base, "avg_frequency", [1, 4], runner=lambda c: S.run(c, ctx))
    for r in rows:
        assert r.error == "" and r.seeds == 1
        assert r.final_ce < math.log(20)  # it learns
        assert r.frames_per_s > 0 and r.speedup > 0
    # repeated runs are bitwise identical
    res1 = S.run(base.with_value("avg_frequency", 1), ctx)
    res1b = S.run(base.with_value("avg_frequency", 1), ctx)
    assert [m.train_ce for m in res1.metrics] == [m.train_ce for m in res1b.metrics]  # deterministic
