"""Host-side logic of the batched engine and the drop policy, on the CPU:
working-cache slot assignment with a per-dialogue kept count (the round cache
keeps staying rounds in place, kept rounds occupy slots [0, n)), the capacity
error, the tier shapes, and the inactivity ledger against the oracle's and the
reference's own ActivityLedger (selection.py:168-204)."""

from __future__ import annotations

import math
import types

import numpy as np
import pytest

from oracle import refkernel
from oracle import rounds as orr


def _stub(K, batch, round_cache=True):
    import paper_2502_15294_b200.decode_engine as de
    s = types.SimpleNamespace()
    s.cfg = types.SimpleNamespace(batch=batch, round_cache=round_cache)
    s.K = K
    s.slot_round = np.full((batch, K), -1, dtype=np.int64)
    s.dialogues = list(range(batch))
    s.assign = lambda kept: de.RoundDecodeEngine.assign_slots(s, kept)
    return s


def test_slots_compact_with_variable_kept_counts():
    pytest.importorskip("torch")
    s = _stub(K=5, batch=2)
    copies = s.assign([[1, 3, 4], [0, 2]])
    assert sorted(copies) == sorted([(0, 0, 1), (0, 1, 3), (0, 2, 4), (1, 0, 0), (1, 1, 2)])
    # dialogue 0 keeps 3 and 4 and adds 6; dialogue 1 shrinks to one round (2 stays only if its slot < 1)
    copies = s.assign([[3, 4, 6, 7], [2]])
    assert set(int(x) for x in s.slot_round[0][:4]) == {3, 4, 6, 7}
    assert int(s.slot_round[0][1]) == 3 and int(s.slot_round[0][2]) == 4      # stayed in place
    assert int(s.slot_round[1][0]) == 2 and all(int(x) == -1 for x in s.slot_round[1][1:])
    assert (1, 0, 2) in copies                                               # moved into slot 0: refetched
    assert all(slot < 4 for b, slot, r in copies if b == 0)


def test_slots_without_round_cache_fetch_everything():
    pytest.importorskip("torch")
    s = _stub(K=2, batch=1, round_cache=False)
    s.assign([[0, 1]])
    copies = s.assign([[0, 1]])
    assert sorted(copies) == [(0, 0, 0), (0, 1, 1)]


def test_slots_capacity_error():
    pytest.importorskip("torch")
    s = _stub(K=2, batch=1)
    with pytest.raises(RuntimeError, match="capacity"):
        s.assign([[0, 1, 2]])


def test_tier_shapes():
    pytest.importorskip("torch")
    from paper_2502_15294_b200.decode_engine import EngineConfig, RoundDecodeEngine
    from paper_2502_15294_b200.selection import SelectionPolicy
    c = EngineConfig(rounds=32, round_tokens=512, decode_steps=128)
    assert RoundDecodeEngine.shapes(c) == dict(K=4, s_lo=32 * 512 + 129, s_up=4 * 512 + 129)
    c = EngineConfig(rounds=32, round_tokens=512, decode_steps=128, policy=SelectionPolicy("adaptive"), max_kept=8)
    assert RoundDecodeEngine.shapes(c)["K"] == 8


def _ledger_runs(cls, window, protect, R, kept_seq):
    led = cls(window=window, protect_recent=protect)
    for r in range(R):
        led.register_round(r, r)
    out = []
    for t, kept in enumerate(kept_seq):
        out.append(sorted(led.update_and_drop(list(kept), R + t, R)))
    return out, sorted(led.active_rounds(R))


@pytest.mark.parametrize("window,protect", [(1, 1), (2, 2), (3, 0), (math.inf, 2)])
def test_activity_ledger_matches_oracle_and_reference(window, protect):
    pytest.importorskip("torch")
    from paper_2502_15294_b200.selection import ActivityLedger
    rng = np.random.default_rng(int(protect * 10 + (0 if math.isinf(window) else window)))
    R = 12
    seq = [sorted(rng.choice(R, size=3, replace=False).tolist()) for _ in range(8)]
    ours = _ledger_runs(ActivityLedger, window, protect, R, seq)
    assert ours == _ledger_runs(orr.ActivityLedger, window, protect, R, seq)
    if refkernel.available():
        ref = refkernel.load_package()
        import importlib
        rsel = importlib.import_module("roundkv.selection")
        assert ours == _ledger_runs(rsel.ActivityLedger, window, protect, R, seq)


def test_step_kernel_config_validation():
    """The answer-loop selector: unknown values are rejected before any
    allocation, and the persistent whole-step kernel (one CTA on every SM) is
    refused for concurrent groups."""
    from paper_2502_15294_b200.decode_engine import EngineConfig, GroupedDecoder, RoundDecodeEngine
    with pytest.raises(ValueError, match="step_kernel"):
        RoundDecodeEngine(EngineConfig(batch=2, step_kernel="fused"), device="cpu")
    with pytest.raises(ValueError, match="groups=1"):
        GroupedDecoder(EngineConfig(batch=4, step_kernel="persistent"), groups=2, device="cpu")
