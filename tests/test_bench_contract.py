"""The bench.py JSON line (the driver's contract): one short run on the GPU
with the extras switched off, every required key present with the right type,
the timing rules honoured (warm-up >= 3, L2 note, clocks sampled under load),
and the roofline / e2e blocks well formed."""
import json
import os
import subprocess
import sys

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu


def test_bench_json_line():
    cmd = [sys.executable, os.path.join(ROOT, "bench.py"), "--steps", "20", "--warmup", "3", "--no-cpu", "--epochs",
           "0", "--no-kron", "--no-cd1", "--e2e-steps", "20", "--per-class", "24"]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]
    d = json.loads(lines[0])
    for k, t in (("metric", str), ("value", float), ("unit", str), ("n_gpus", int), ("steps", int),
                 ("warmup", int), ("ms_per_step", float), ("higher_is_better", bool), ("scaling", str),
                 ("dtype", str), ("data", str), ("config", dict), ("clocks", dict), ("gpu_launches", int),
                 ("roofline", dict), ("e2e", dict)):
        assert isinstance(d[k], t), (k, type(d[k]))
    assert d["n_gpus"] == 1 and d["steps"] == 20 and d["warmup"] == 3 and d["higher_is_better"] is True
    assert d["scaling"] == "weak" and "vs_baseline" in d and d["value"] > 0 and d["ms_per_step"] > 0
    assert d["config"]["workload"] and "l2" in d["config"]
    r = d["roofline"]
    assert r["bound"] in ("tensor", "hbm") and r["unit"] in ("TFLOP/s", "GB/s")
    assert 0 < r["achieved"] and 0 < r["peak"] and abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-9
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    c = d["clocks"]
    assert c["samples"] > 0 and c["sm_mhz"] > 0 and isinstance(c["reasons"], list)
    assert d["gpu_launches"] > 0
