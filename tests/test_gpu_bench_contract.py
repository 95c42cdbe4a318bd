"""bench.py's JSON line (the driver's contract), from a short run on the GPU: one line on stdout
with the metric, the roofline object of the dominant kernel, e2e, clocks and launch count."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_bench_json_line_contract():
    r = subprocess.run([sys.executable, "bench.py", "--steps", "16", "--warmup", "3", "--graph-steps", "8",
                        "--e2e-steps", "1", "--no-cpu-baseline"], cwd=ROOT, capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.strip()]
    assert len(lines) == 1, r.stdout[-2000:]
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "roofline", "clocks", "gpu_launches", "e2e"):
        assert k in d, k
    assert d["n_gpus"] == 1 and d["steps"] == 16 and d["warmup"] >= 3 and d["value"] > 0
    assert d["gpu_launches"] == 5 * 16  # lookup, choose-k, scan, race, emit (+alpha update CTA) per step
    rf = d["roofline"]
    assert rf["bound"] == "hbm" and rf["unit"] == "GB/s" and 0 < rf["frac"] < 1
    assert abs(rf["frac"] - rf["achieved"] / rf["peak"]) < 1e-9
    assert rf["traffic"] is None or rf["traffic"] > 0.9 * rf["alg_bytes_per_launch"]
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    assert "workload" in d["config"] and "l2_defeat" in d["config"]
    # every other workload as a sub-object, each timed with its own roofline, clocks and device status
    w = d["workloads"]
    for name in ("config4", "config4_sharded_p2p", "greedy", "logits", "config5", "loop"):
        sub = w[name]
        assert "error" not in sub, (name, sub)
        assert sub["value"] > 0 and sub["ms_per_step"] > 0, name
        assert sub["roofline"]["peak"] > 0 and 0 < sub["roofline"]["frac"] < 1.5, name
        assert "sm_mhz" in sub["clocks"], name
        assert sub["device_status"] in (0, None), name
    assert w["config4"]["config"]["vocab"] == 128256
