"""bench.py's reference arm on CPU: the JSON line the driver reads (metric,
unit, impl, cpu_baseline, e2e with zero copies), timed inside one oracle run
from the oracle's per-generation stamps (a positive, finite window)."""

import json
import math
import os
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_line():
    res = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--steps", "2", "--warmup", "3"],
                         capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert res.returncode == 0, res.stderr[-2000:]
    lines = [ln for ln in res.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["unit"] == "domain-evals/s" and d["higher_is_better"] is True
    assert d["steps"] == 2 and d["warmup"] == 3 and d["n_gpus"] == 1
    assert math.isfinite(d["value"]) and 0 < d["value"] < 1e13  # a real CPU rate, not a clamped window
    assert d["ms_per_step"] > 0.1
    assert d["cpu_baseline"]["kind"] == "port" and d["cpu_baseline"]["value"] == d["value"]
    assert d["cpu_baseline"]["cores"] >= 1 and "sample" in d["cpu_baseline"]
    assert d["e2e"] == {"value": d["value"], "unit": d["unit"], "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}
    assert d["config"]["timed_generations"] == [4, 5]


def test_oracle_generation_stamps():
    from oracle import oracle as O
    from paper_2511_01255_b200 import tables as T

    t = T.build_tables("thg", 1.0, 600, (0.3, 0.7))
    P = O.Problem("thg", t.e1[None], t.b[None], np.array([t.w]), np.array([t.hconst]), t.normalization)
    stamps = np.zeros(21)
    trace, *_ = O.run(P, "hybrid", 16, 20, 1, stop_after=8, gen_end_s=stamps)
    plain, *_ = O.run(P, "hybrid", 16, 20, 1, stop_after=8)
    assert np.array_equal(trace, plain)  # stamping does not change the run
    assert np.all(np.diff(stamps[:9]) >= 0) and stamps[0] > 0 and np.all(stamps[9:] == 0)


@pytest.mark.gpu
def test_gpu_line_contract():
    """The device arm's JSON line: the keys the driver and the judge read."""
    res = subprocess.run([sys.executable, "bench.py", "--steps", "3", "--warmup", "3", "--no-cpu-baseline"],
                         capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert res.returncode == 0, res.stderr[-3000:]
    lines = [ln for ln in res.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "roofline", "e2e", "clocks", "gpu_launches"):
        assert k in d, k
    assert d["steps"] == 3 and d["warmup"] == 3 and d["n_gpus"] == 1 and d["higher_is_better"] is True
    assert d["value"] > 1e10 and d["gpu_launches"] > 0 and "workload" in d["config"]
    r = d["roofline"]
    assert r["bound"] in ("hbm", "fp64", "tensor") and 0 < r["frac"] <= 1.5 and r["achieved"] > 0 and r["peak"] > 0
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    assert d["clocks"]["sm_mhz"] > 0
