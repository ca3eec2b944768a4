"""The reference's OWN turn loop running on this package (SURVEY.md §8b
[verified] recipe): the unmodified reference package (`roundkv`, staged into
oracle/_ref by `make -C oracle ref`) drives `RoundPipeline.run_turn`
(pipeline.py:192-394) on its NumPy model, with every hot-path entry point
replaced by this package:

  * `roundkv.engine.attention_forward` (bound at engine.py:20)  -> librk
    (`paper_2502_15294_b200.backend.attention_forward`, the kernel contract);
  * `roundkv.pipeline.{aggregate_round_attention, normalize, select}`
    (bound at pipeline.py:32-49)                                 -> device Eq. 1 +
    bit-exact device selection;
  * the tiered store, injected through `store=` (pipeline.py:120,139-142) ->
    `NumpyViewStore` (physical pinned-host / device tiers, rk_h2d_gather).

The C1 conversation must reproduce the reference's golden turns (answers,
kept rounds, raw masses, transfer ledger).  A second test applies
INTEGRATION.md's `backend.py` branch (ROUNDKV_BACKEND=cuda) to a scratch copy
of the reference package and runs the same loop through it.
"""

from __future__ import annotations

import json
import os
import shutil
import subprocess
import sys

import numpy as np
import pytest

from conftest import GOLDEN, REPO

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

from oracle import refkernel  # noqa: E402

if not refkernel.available():  # pragma: no cover
    pytest.skip("reference package not staged (make -C oracle ref)", allow_module_level=True)


def _check_turn(z, t, res):
    m = res.metrics
    assert tuple(int(x) for x in m.kept) == tuple(int(x) for x in z[f"t{t}_kept"]), t
    if f"t{t}_raw" in z.files:
        np.testing.assert_allclose(np.asarray(m.distribution.raw), z[f"t{t}_raw"], rtol=1e-5)
        np.testing.assert_allclose(np.asarray(m.distribution.masses), z[f"t{t}_masses"], rtol=1e-5)
    led = z[f"t{t}_ledger"]
    assert [m.upper_h2d_events, m.upper_h2d_bytes, m.lower_h2d_events, m.lower_h2d_bytes,
            m.d2h_events, m.d2h_bytes, m.device_used_peak, m.hist_tokens, m.hist_tokens_attended,
            m.selection_invocations] == led.tolist(), t
    assert [int(x) for x in res.answer_ids] == [int(x) for x in z[f"t{t}_answer"]], t


def test_reference_run_turn_on_librk(monkeypatch):
    rk = refkernel.load_package()
    import roundkv.engine as reng
    import roundkv.pipeline as rpipe
    import roundkv.selection as rsel

    from paper_2502_15294_b200 import backend, selection, stats
    from paper_2502_15294_b200.store import NumpyViewStore

    assert rk.__file__.startswith(str(REPO / "oracle" / "_ref"))
    calls = {"attn": 0, "select": 0}

    def attn(*a, **kw):
        calls["attn"] += 1
        return backend.attention_forward(*a, **kw)

    def sel(*a, **kw):
        calls["select"] += 1
        return selection.select(*a, **kw)

    monkeypatch.setattr(reng, "attention_forward", attn)
    monkeypatch.setattr(rpipe, "aggregate_round_attention", stats.aggregate_round_attention)
    monkeypatch.setattr(rpipe, "normalize", stats.normalize)
    monkeypatch.setattr(rpipe, "select", sel)

    z = np.load(GOLDEN / "c1_pipeline.npz")
    model = reng.Model(reng.ModelConfig(num_layers=4, num_heads=8, d_model=512, rng_seed=42))
    store = NumpyViewStore(4, 2, 512)
    pipe = rpipe.RoundPipeline(model, 2, policy=rsel.SelectionPolicy("top_percent", fraction=0.10), store=store)
    for t in range(int(z["turns"])):
        res = pipe.run_turn(list(z["questions"][t]), max_decode_steps=int(z["steps"]))
        _check_turn(z, t, res)
        assert isinstance(res.metrics.distribution, stats.RoundDistribution) or t == 0
    # every attention call and every selection went through this package
    assert calls["attn"] > 0 and calls["select"] == int(z["turns"]) - 1
    pipe.end_session()
    assert store.device_used_bytes == 0


BACKEND_BRANCH = '''elif _requested == "cuda":
    from paper_2502_15294_b200 import backend as _cuda   # librk.so, sm_100a (INTEGRATION.md §1)
    _impl = _cuda
'''

SCRIPT = r"""
import json, sys
import numpy as np
sys.path.insert(0, sys.argv[1]); sys.path.insert(0, sys.argv[2])
import roundkv, roundkv.engine as reng, roundkv.pipeline as rpipe, roundkv.selection as rsel
from paper_2502_15294_b200.store import NumpyViewStore
assert roundkv.BACKEND_NAME == "cuda", roundkv.BACKEND_NAME
assert reng.attention_forward.__module__ == "paper_2502_15294_b200.backend"
z = np.load(sys.argv[3])
model = reng.Model(reng.ModelConfig(num_layers=4, num_heads=8, d_model=512, rng_seed=42))
pipe = rpipe.RoundPipeline(model, 2, policy=rsel.SelectionPolicy("top_percent", fraction=0.10),
                           store=NumpyViewStore(4, 2, 512))
out = []
for t in range(int(sys.argv[4])):
    res = pipe.run_turn(list(z["questions"][t]), max_decode_steps=int(z["steps"]))
    out.append({"answer": [int(x) for x in res.answer_ids], "kept": [int(x) for x in res.metrics.kept]})
print(json.dumps({"backend": roundkv.BACKEND_NAME, "turns": out}))
"""


def test_reference_backend_cuda_branch(tmp_path):
    """the reference's backend.py with the added `cuda`
    branch selects librk at import (ROUNDKV_BACKEND=cuda); the reference's
    turn loop then reproduces its own golden answers on it."""
    pkg = tmp_path / "roundkv"
    shutil.copytree(refkernel.REF_DIR, pkg)
    src = (pkg / "backend.py").read_text()
    anchor = 'elif _requested == "auto":'
    assert anchor in src
    (pkg / "backend.py").write_text(src.replace(anchor, BACKEND_BRANCH + anchor, 1))
    turns = 4
    env = dict(os.environ, ROUNDKV_BACKEND="cuda")
    res = subprocess.run([sys.executable, "-c", SCRIPT, str(tmp_path), str(REPO), str(GOLDEN / "c1_pipeline.npz"),
                          str(turns)], capture_output=True, text=True, timeout=600, env=env)
    assert res.returncode == 0, res.stderr[-3000:]
    out = json.loads(res.stdout.strip().splitlines()[-1])
    assert out["backend"] == "cuda"
    z = np.load(GOLDEN / "c1_pipeline.npz")
    for t in range(turns):
        assert out["turns"][t]["kept"] == [int(x) for x in z[f"t{t}_kept"]], t
        assert out["turns"][t]["answer"] == [int(x) for x in z[f"t{t}_answer"]], t
