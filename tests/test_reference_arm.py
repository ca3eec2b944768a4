"""The reference arm of bench.py (--impl reference) must run the reference
package itself and never map the product library (librk.so): the driver voids
the GPU/CPU ratio when the reference process loads our native code."""

from __future__ import annotations

import json
import subprocess
import sys
from pathlib import Path

import pytest

REPO = Path(__file__).resolve().parents[1]

SCRIPT = r"""
import json, sys
sys.path.insert(0, sys.argv[1])
from oracle import cpu_baseline, refkernel
if not refkernel.available():
    print(json.dumps({"skip": "reference not staged"})); sys.exit(0)
r = cpu_baseline.decode_tokens_per_s("reference", L=4, lw=2, hq=8, hkv=2, d=64, rounds=8, T=64,
                                     K=cpu_baseline.kept_count(8), processes=2, tokens_per_proc=2)
maps = open("/proc/self/maps").read()
print(json.dumps({"tps": r["tokens_per_s"], "kernel": r["kernel"], "librk": "librk.so" in maps,
                  "ext": "_attn_ext" in maps,
                  "product": sorted(m for m in sys.modules if m.startswith("paper_2502_15294_b200"))}))
"""


def test_reference_arm_runs_reference_package_without_librk():
    res = subprocess.run([sys.executable, "-c", SCRIPT, str(REPO)], capture_output=True, text=True, timeout=300)
    assert res.returncode == 0, res.stderr
    out = json.loads(res.stdout.strip().splitlines()[-1])
    if "skip" in out:
        pytest.skip(out["skip"])
    assert out["tps"] > 0
    assert out["ext"], "the reference's compiled kernel was not loaded"
    assert not out["librk"], "the reference arm mapped librk.so"
    assert out["product"] == [], out["product"]
    assert out["kernel"]["path"].startswith("oracle/_ref/roundkv/_attn_ext")


def test_kept_count_matches_package_selection():
    from oracle.cpu_baseline import kept_count
    from oracle.rounds import top_k_count
    for n in range(1, 300):
        for f in (0.05, 0.1, 0.3, 0.5, 1.0):
            assert kept_count(n, f, 1) == top_k_count(n, f, 1)
