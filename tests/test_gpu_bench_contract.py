"""bench.py's one-line JSON contract on a short run (C3 workload, 1 timed step,
3 warm-up steps, 2 videos, T = 20, no secondary lines): every key the driver
and the judge read is present with the right type, the headline is the
whole-job videos/s, and the e2e, roofline, clocks and launch-count claims are
well formed.  (The CPU-baseline leg is exercised by the reference-arm test.)"""

import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(args, timeout=900):
    out = subprocess.run([sys.executable, "bench.py"] + args, cwd=ROOT, capture_output=True,
                         text=True, timeout=timeout)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.strip().splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]
    return json.loads(lines[0])


def test_ours_line_contract(cuda_dev):
    d = _run(["--workload", "c3", "--steps", "1", "--warmup", "3", "--videos", "2",
              "--timesteps", "20", "--no-extra", "--no-cpu-baseline"])
    for k, t in (("metric", str), ("value", float), ("unit", str), ("n_gpus", int),
                 ("steps", int), ("warmup", int), ("ms_per_step", float),
                 ("higher_is_better", bool), ("scaling", str), ("dtype", str), ("data", str),
                 ("config", dict), ("roofline", dict), ("e2e", dict), ("gpu_launches", int),
                 ("clocks", dict)):
        assert isinstance(d[k], t), (k, d.get(k))
    assert d["metric"] == "videos_per_s" and d["unit"] == "videos/s"
    assert d["n_gpus"] == 1 and d["steps"] == 1 and d["warmup"] == 3 and d["value"] > 0
    assert d["vs_baseline"] is None and d["scaling"] == "weak"
    assert "workload" in d["config"]
    r = d["roofline"]
    assert r["bound"] in ("hbm", "tensor") and r["unit"] in ("GB/s", "TOP/s", "TFLOP/s")
    assert 0 < r["frac"] < 1 and abs(r["achieved"] / r["peak"] - r["frac"]) < 1e-9
    e = d["e2e"]
    assert e["unit"] == "videos/s" and e["value"] > 0
    assert e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    assert d["gpu_launches"] > 100
    assert {"sm_mhz", "sm_max_mhz", "reasons"} <= set(d["clocks"])


def test_reference_line_contract(cuda_dev):
    d = _run(["--impl", "reference", "--workload", "c3", "--steps", "1", "--warmup", "1"])
    assert d["impl"] == "reference" and d["metric"] == "videos_per_s" and d["value"] > 0
    cb = d["cpu_baseline"]
    assert cb["kind"] in ("reference", "port") and cb["cores"] >= 1 and cb["sample"]
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
