"""bench.py's JSON line keeps the driver's contract (one line; the metric,
roofline, e2e, clocks and launch-count keys; device-timed and end-to-end
throughput both positive) on a small C2-shaped run."""

from __future__ import annotations

import json
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

REPO = Path(__file__).resolve().parents[1]


def test_bench_json_contract():
    cmd = [sys.executable, str(REPO / "bench.py"), "--batch", "2", "--decode-steps", "4", "--steps", "3",
           "--warmup", "3", "--no-cpu", "--no-fetch-all", "--host-unique", "1"]
    res = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=REPO)
    assert res.returncode == 0, res.stderr[-2000:]
    lines = [ln for ln in res.stdout.splitlines() if ln.strip()]
    assert len(lines) == 1, lines
    d = json.loads(lines[0])
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
                "scaling", "vs_baseline", "dtype", "data", "config", "roofline", "e2e", "clocks", "gpu_launches",
                "k_boundary", "gpu_kv_saved"):
        assert key in d, key
    assert d["n_gpus"] == 1 and d["steps"] == 3 and d["warmup"] == 3 and d["scaling"] == "weak"
    assert d["value"] > 0 and d["higher_is_better"] is True and d["vs_baseline"] is None
    assert "workload" in d["config"]
    r = d["roofline"]
    for key in ("bound", "achieved", "peak", "unit", "frac", "traffic"):
        assert key in r, key
    assert r["bound"] == "hbm" and r["unit"] == "GB/s" and 0 < r["frac"] < 1.5
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    for key in ("sm_mhz", "sm_max_mhz", "reasons"):
        assert key in d["clocks"], key
    assert d["gpu_launches"] > 0
    assert d["gpu_kv_saved"]["saved_frac"] > 0.54          # north star: >= 54 % of full-cache KV saved
