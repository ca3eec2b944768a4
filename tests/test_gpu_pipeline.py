"""GPU drop-in pipeline vs the REAL reference: the C1 tiny config
(Model(4 layers, 8 heads, d_model 512, seed 42), watershed 2,
top_percent 0.10, 63 random byte ids per question, 63 decode steps) must
reproduce the reference's kept rounds, raw masses, answer ids and transfer
ledger turn by turn (tests/golden/c1_pipeline.npz, tools/make_golden.py)."""

from __future__ import annotations

import numpy as np
import pytest

from conftest import GOLDEN, load_store_cases

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2502_15294_b200 import store as st  # noqa: E402
from paper_2502_15294_b200.engine import Model, ModelConfig  # noqa: E402
from paper_2502_15294_b200.errors import CapacityError, ConsistencyError, DomainError  # noqa: E402
from paper_2502_15294_b200.pipeline import RoundPipeline  # noqa: E402
from paper_2502_15294_b200.selection import SelectionPolicy  # noqa: E402


def test_c1_pipeline_matches_reference():
    z = np.load(GOLDEN / "c1_pipeline.npz")
    model = Model(ModelConfig(num_layers=4, num_heads=8, d_model=512, rng_seed=42))
    pipe = RoundPipeline(model, 2, policy=SelectionPolicy("top_percent", fraction=0.10))
    agree = 0
    for t in range(int(z["turns"])):
        res = pipe.run_turn(list(z["questions"][t]), max_decode_steps=int(z["steps"]))
        m = res.metrics
        assert m.kept == tuple(z[f"t{t}_kept"]), t
        if f"t{t}_raw" in z.files:
            np.testing.assert_allclose(m.distribution.raw, z[f"t{t}_raw"], rtol=1e-5)
        led = z[f"t{t}_ledger"]
        assert [m.upper_h2d_events, m.upper_h2d_bytes, m.lower_h2d_events, m.lower_h2d_bytes,
                m.d2h_events, m.d2h_bytes, m.device_used_peak, m.hist_tokens, m.hist_tokens_attended,
                m.selection_invocations] == led.tolist(), t
        want = list(z[f"t{t}_answer"])
        assert res.answer_ids == want, (t, res.answer_ids[:10], want[:10])
        agree += 1
    assert agree == int(z["turns"])


def test_mask_mode_equals_splice():
    """attend_mode='mask' (full assembly + restricted visibility) == splice (pipeline.py:271-280)."""
    model = Model(ModelConfig(num_layers=4, num_heads=4, d_model=64, rng_seed=3))
    rng = np.random.default_rng(5)
    qs = [list(rng.integers(0, 256, size=9)) for _ in range(4)]
    a = RoundPipeline(model, 2, policy=SelectionPolicy("top_percent", fraction=0.3))
    b = RoundPipeline(model, 2, policy=SelectionPolicy("top_percent", fraction=0.3))
    b.attend_mode = "mask"
    for q in qs:
        ra, rb = a.run_turn(q, 8), b.run_turn(q, 8)
        assert ra.answer_ids == rb.answer_ids
        assert ra.metrics.kept == rb.metrics.kept


def test_all_policy_equals_baseline():
    """policy 'all' answers == full-cache baseline (SPEC acceptance 2)."""
    model = Model(ModelConfig(num_layers=4, num_heads=4, d_model=64, rng_seed=9))
    rng = np.random.default_rng(6)
    qs = [list(rng.integers(0, 256, size=7)) for _ in range(3)]
    a = RoundPipeline(model, 2, policy=SelectionPolicy("all"))
    b = RoundPipeline.baseline(model, 2)
    for q in qs:
        assert a.run_turn(q, 6).answer_ids == b.run_turn(q, 6).answer_ids


def _apply(store, op, d, lw, L):
    kind = op[0]
    if kind == "put":
        store.put_round(op[1], np.zeros((lw, 2, op[2], d), np.float32), np.zeros((L - lw, 2, op[2], d), np.float32),
                        np.arange(op[2]), upper_on_device=op[3])
    elif kind == "begin":
        store.begin_turn(op[1])
    elif kind == "fetch_upper":
        store.fetch_upper(op[1])
    elif kind == "fetch_lower_all":
        store.fetch_lower_all(op[1])
    elif kind == "writeback_upper":
        store.writeback_upper(op[1])
    elif kind == "drop_upper":
        store.drop_upper(op[1])
    else:
        store.end_session()


def test_tiered_store_ledger_matches_reference():
    data = load_store_cases()
    for seq in data["sequences"]:
        s = st.TieredStore(seq["L"], seq["lw"], seq["d"], device_capacity=seq["cap"],
                           evict_lower_on_pressure=seq["evict"])
        for op, res in zip(seq["ops"], seq["results"]):
            err = None
            try:
                _apply(s, op, seq["d"], seq["lw"], seq["L"])
            except (ConsistencyError, CapacityError, DomainError) as e:
                err = type(e).__name__
            assert err == res["err"], (op, res)
            assert s.device_used_bytes == res["used"]
            led = s.ledger
            assert [led.h2d_events, led.h2d_bytes, led.d2h_events, led.d2h_bytes] == res["ledger"]
            assert led.report_rows() == res["per_turn"]
            assert {f"{k[0]}:{k[1]}": b.tier for k, b in s.blocks.items()} == res["tiers"]
            for b in s.blocks.values():           # tiers are physical
                if b.tier == "device":
                    assert b.payload.is_cuda
                elif b.tier == "host":
                    assert not b.payload.is_cuda and b.payload.is_pinned()


def test_fetch_upper_moves_bytes():
    s = st.TieredStore(4, 2, 8)
    up = torch.randn(2, 2, 5, 8)
    s.put_round(0, torch.randn(2, 2, 5, 8), up, np.arange(5))
    s.begin_turn(1)
    blocks = s.fetch_upper([0])
    torch.cuda.synchronize()
    assert blocks[0].payload.is_cuda
    torch.testing.assert_close(blocks[0].payload.cpu(), up)
    assert s.ledger.per_turn[-1].h2d_events == 1


@pytest.mark.parametrize("name,kw", [
    ("drop2", dict(policy=SelectionPolicy("top_percent", fraction=0.25), drop_window=2, drop_protect=1)),
    ("fixed", dict(policy=SelectionPolicy("fixed", v=0.12))),
    ("adaptive", dict(policy=SelectionPolicy("adaptive", kappa=0.5))),
    ("pre", dict(policy=SelectionPolicy("top_percent", fraction=0.25))),    # capture_mode="pre" model
    ("baseline", dict(mode="baseline")),                                    # full-cache baseline mode
    ("mask", dict(policy=SelectionPolicy("top_percent", fraction=0.25))),   # attend_mode="mask"
])
def test_c1_policy_and_drop_variants_match_reference(name, kw):
    """Inactivity drop policy (ActivityLedger.update_and_drop + store.drop_upper,
    selection.py:168-204, store.py:280-285), the fixed / adaptive strategies and
    the head-summed-logit capture (capture_mode="pre", engine.py:187-200)
    through whole turns: kept rounds, dropped set, answers and transfer ledger
    equal the reference's (tests/golden/c1_variants.npz)."""
    z = np.load(GOLDEN / "c1_variants.npz")
    model = Model(ModelConfig(num_layers=4, num_heads=8, d_model=512, rng_seed=42,
                              capture_mode="pre" if name == "pre" else "post"))
    pipe = RoundPipeline(model, 2, **kw)
    if name == "mask":
        pipe.attend_mode = "mask"
    for t in range(6):
        res = pipe.run_turn(list(z[f"{name}_t{t}_q"]), max_decode_steps=15)
        m = res.metrics
        assert m.kept == tuple(z[f"{name}_t{t}_kept"]), (name, t)
        assert sorted(pipe.activity.dropped) == list(z[f"{name}_t{t}_dropped"]), (name, t)
        assert list(res.answer_ids) == list(z[f"{name}_t{t}_answer"]), (name, t)
        assert [m.upper_h2d_events, m.upper_h2d_bytes, m.d2h_events, m.d2h_bytes, m.device_used_peak,
                m.hist_tokens_attended] == z[f"{name}_t{t}_ledger"].tolist(), (name, t)
