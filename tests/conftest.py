"""Shared fixtures.  `gpu` marks tests that need a B200 (`pytest -m gpu`);
everything else runs on the CPU build container (`pytest -m "not gpu"`)."""

from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np
import pytest

REPO = Path(__file__).resolve().parents[1]
GOLDEN = REPO / "tests" / "golden"
if str(REPO) not in sys.path:
    sys.path.insert(0, str(REPO))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")


def load_kernel_cases():
    z = np.load(GOLDEN / "kernel_cases.npz")
    cases = []
    for i in range(int(z["count"])):
        p = f"c{i}_"
        c = {}
        for name in ("q", "k", "v"):
            if p + name + "_bf16" in z.files:
                c[name] = (z[p + name + "_bf16"].astype(np.uint32) << 16).view(np.float32)
                c["bf16"] = True
            else:
                c[name] = z[p + name]
                c["bf16"] = False
        c["q_pos"], c["k_pos"] = z[p + "q_pos"], z[p + "k_pos"]
        c["allowed"] = z[p + "allowed"] if bool(z[p + "masked"]) else None
        c["capture"] = bool(z[p + "capture"])
        c["out"] = z[p + "out"]
        c["scores"] = z[p + "scores"] if c["capture"] else None
        cases.append(c)
    return cases


def load_stats_cases():
    z = np.load(GOLDEN / "stats_cases.npz")
    out = []
    for i in range(int(z["count"])):
        p = f"s{i}_"
        out.append({k[len(p):]: z[k] for k in z.files if k.startswith(p)})
    return out


def load_select_cases():
    cases = json.loads((GOLDEN / "select_cases.json").read_text())
    for c in cases:
        c["raw"] = np.array([float.fromhex(x) for x in c["raw"]])
        c["masses"] = np.array([float.fromhex(x) for x in c["masses"]])
    return cases


def load_store_cases():
    return json.loads((GOLDEN / "store_cases.json").read_text())


@pytest.fixture
def rng():
    return np.random.default_rng(1234)


def cuda_available() -> bool:
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False
