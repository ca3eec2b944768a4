"""The N>1 product path on one GPU: bench.py under torchrun with two ranks
sharing the device (RK_SHARE_GPU=1, gloo barrier) serves the same dialogues as
one process, each rank its round-robin shard with no data-path collective, and
every dialogue keeps the same rounds as in the single-process run (the data and
questions of a dialogue are seeded by its global id)."""

from __future__ import annotations

import json
import os
import socket
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

REPO = Path(__file__).resolve().parents[1]
FLAGS = ["--steps", "2", "--warmup", "3", "--no-cpu", "--no-e2e", "--no-fetch-all", "--decode-steps", "8",
         "--host-unique", "0"]


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _line(cmd, env=None):
    res = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=REPO, env=env)
    assert res.returncode == 0, res.stderr[-3000:]
    lines = [ln for ln in res.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, res.stdout[-2000:]
    return json.loads(lines[0])


def test_two_ranks_on_one_gpu_match_one_process():
    one = _line([sys.executable, str(REPO / "bench.py"), "--batch", "4"] + FLAGS)
    env = dict(os.environ, RK_SHARE_GPU="1")
    two = _line([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                 "--master-addr", "127.0.0.1", "--master-port", str(_port()), str(REPO / "bench.py"), "--gpus", "2",
                 "--batch", "2"] + FLAGS, env=env)
    assert one["n_gpus"] == 1 and two["n_gpus"] == 2
    assert two["config"]["global_batch"] == 4 and two["scaling"] == "weak"
    assert sorted(one["kept_by_dialogue"]) == sorted(two["kept_by_dialogue"]) == ["0", "1", "2", "3"]
    assert one["kept_by_dialogue"] == two["kept_by_dialogue"]
    assert two["value"] > 0 and two["ms_per_step"] > 0
