"""Pin the CPU oracle to the real reference: every golden vector produced by
`tools/make_golden.py` (reference imported in the build container) must be
reproduced by `oracle/` — bit-exact for indices, ledgers and the memory model,
within 1e-12 relative for fp64 attention arithmetic."""

from __future__ import annotations

import numpy as np
import pytest

from conftest import GOLDEN, load_kernel_cases, load_select_cases, load_stats_cases, load_store_cases
from oracle import attention as oatt
from oracle import rounds as orr
from oracle.model import Model, ModelConfig, Pipeline
from paper_2502_15294_b200.errors import ConsistencyError, CapacityError, DomainError, InvariantError

KERNEL = load_kernel_cases()


@pytest.mark.parametrize("idx", range(len(KERNEL)))
def test_attention_oracle_matches_reference(idx):
    c = KERNEL[idx]
    out, scores = oatt.attention_forward(c["q"], c["k"], c["v"], c["q_pos"], c["k_pos"],
                                         allowed=c["allowed"], capture=c["capture"])
    np.testing.assert_allclose(out, c["out"], rtol=1e-6, atol=1e-6)
    if c["capture"]:
        np.testing.assert_allclose(scores, c["scores"], rtol=1e-12, atol=1e-14)
    else:
        assert scores is None


def test_attention_oracle_contract_errors(rng):
    q = rng.standard_normal((5, 4, 8)).astype(np.float32)
    k = rng.standard_normal((12, 4, 8)).astype(np.float32)
    with pytest.raises(InvariantError, match="no visible key"):
        oatt.attention_forward(q, k, k, np.arange(7, 12), np.arange(12), allowed=np.zeros(12, bool))
    with pytest.raises(DomainError):
        oatt.attention_forward(q, k, k[:, :2], np.arange(7, 12), np.arange(12))
    with pytest.raises(DomainError):
        oatt.attention_forward(q, k, k, np.arange(2), np.arange(12))
    out, sc = oatt.attention_forward(q[:0], k, k, np.zeros(0, np.int64), np.arange(12), capture=True)
    assert out.shape == (0, 32) and sc.shape == (0, 12)


def test_gqa_oracle_is_expansion(rng):
    q = rng.standard_normal((3, 8, 16)).astype(np.float32)
    k = rng.standard_normal((20, 2, 16)).astype(np.float32)
    v = rng.standard_normal((20, 2, 16)).astype(np.float32)
    out, sc = oatt.attention_forward_gqa(q, k, v, np.arange(17, 20), np.arange(20), capture=True)
    ke, ve = np.repeat(k, 4, axis=1), np.repeat(v, 4, axis=1)
    out2, sc2 = oatt.attention_forward(q, ke, ve, np.arange(17, 20), np.arange(20), capture=True)
    np.testing.assert_array_equal(out, out2)
    np.testing.assert_array_equal(sc, sc2)


def test_pairwise_sum_is_numpy_order(rng):
    for _ in range(400):
        n = int(rng.integers(0, 600))
        a = rng.random(n) * 10.0 ** rng.uniform(-8, 8, size=n)
        assert orr.np_pairwise_sum(a) == a.sum()
        if n:
            m, s = orr.np_mean_std(a)
            assert m == a.mean() and s == a.std()


@pytest.mark.parametrize("case", load_stats_cases(), ids=lambda c: "s")
def test_aggregate_and_normalize_match_reference(case):
    rounds = orr.make_rounds([tuple(x) for x in case["layout"]])
    n = len(rounds) - 1
    raw = orr.aggregate_round_attention(case["scores"], rounds, "question", n,
                                        active_rounds=list(case["active"]),
                                        row_offset=int(case["row_offset"]))
    np.testing.assert_array_equal(raw, case["raw"])
    dist = orr.normalize(raw, round_indices=list(case["active"]))
    np.testing.assert_array_equal(dist.masses, case["masses"])
    assert dist.degenerate == bool(case["degenerate"])


def test_selection_matches_reference_bit_exact():
    cases = load_select_cases()
    assert len(cases) > 100
    for c in cases:
        dist = orr.normalize(c["raw"])
        np.testing.assert_array_equal(dist.masses, c["masses"])
        assert dist.degenerate == c["degenerate"]
        for r in c["results"]:
            pol = orr.SelectionPolicy(kind=r["kind"], **r["params"])
            assert list(orr.select(dist, pol)) == r["kept"], (r, c["raw"][:8])


def test_spec_selection_examples():
    # SPEC.md:280-299 examples, re-verified against the code in SURVEY §8c
    d = orr.normalize(np.array([.5, .05, .3, .15]))
    assert orr.select(d, orr.SelectionPolicy("fixed", v=0.1)) == (0, 2, 3)
    d = orr.normalize(np.full(20, 1.0))
    assert orr.select(d, orr.SelectionPolicy("fixed", v=0.1)) == (0,)
    assert orr.top_k_count(30, 0.1, 1) == 3 and orr.top_k_count(5, 0.1, 1) == 1
    d = orr.normalize(np.array([.7, .1, .1, .1]))
    assert orr.select(d, orr.SelectionPolicy("adaptive", kappa=1.0)) == (0,)
    d = orr.normalize(np.array([.3, .2, .3, .2]))
    assert orr.select(d, orr.SelectionPolicy("top_percent", fraction=0.5)) == (0, 2)


def _apply_store_op(store, op):
    kind = op[0]
    if kind == "put":
        store.put_round(op[1], op[2], upper_on_device=op[3])
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


def test_store_ledger_matches_reference():
    data = load_store_cases()
    for seq in data["sequences"]:
        st = orr.StoreModel(seq["L"], seq["lw"], seq["d"], device_capacity=seq["cap"],
                            evict_lower_on_pressure=seq["evict"])
        for op, res in zip(seq["ops"], seq["results"]):
            err = None
            try:
                _apply_store_op(st, op)
            except (ConsistencyError, CapacityError, DomainError) as e:
                err = type(e).__name__
            assert err == res["err"], (op, res)
            assert st.used == res["used"]
            led = st.ledger
            assert [led.h2d_events, led.h2d_bytes, led.d2h_events, led.d2h_bytes] == res["ledger"]
            assert led.rows() == res["per_turn"]
            assert {f"{k[0]}:{k[1]}": t for k, t in st.tier.items()} == res["tiers"]


def test_memory_model_matches_reference():
    data = load_store_cases()
    for m in data["memory"]:
        if "args" in m:
            L, lw, K, T = m["args"]
            assert orr.memory_ratio(L, lw, K, T) == float.fromhex(m["ratio"])
            assert orr.save_percent(L, lw) == m["save"]
            fp = orr.footprint_report(1, 1024, 4096, L, lw, K, T)
            for key, val in m["fp"].items():
                want = float.fromhex(val) if isinstance(val, str) else val
                assert fp[key] == want
        else:
            L, lw = m["table5"]
            assert orr.save_percent(L, lw) == m["save"] == m["published"]


def test_c1_pipeline_oracle_matches_reference():
    """C1 tiny whole-turn parity of the oracle's run_turn restatement."""
    z = np.load(GOLDEN / "c1_pipeline.npz")
    model = Model(ModelConfig(num_layers=4, num_heads=8, d_model=512, rng_seed=42))
    pipe = Pipeline(model, 2, orr.SelectionPolicy("top_percent", fraction=0.10))
    turns = int(z["turns"])
    for t in range(min(turns, 4)):       # first 4 turns keep the CPU suite fast
        res = pipe.run_turn(list(z["questions"][t]), max_decode_steps=int(z["steps"]))
        assert res["answer_ids"] == list(z[f"t{t}_answer"])
        assert res["kept"] == tuple(z[f"t{t}_kept"])
        if res["raw"] is not None:
            np.testing.assert_allclose(res["raw"], z[f"t{t}_raw"], rtol=1e-9)
        rec = pipe.store.ledger.per_turn[-1]
        led = z[f"t{t}_ledger"]
        assert rec.h2d_bytes == led[1] + led[3]
        assert rec.d2h_bytes == led[5]


# ----------------------------------------------------------------- calibration (stats.py:118-181)
def _calib():
    return np.load(GOLDEN / "calib_cases.npz")


def test_oracle_kl_curve_and_watershed_match_reference():
    z = _calib()
    curves = []
    for i in range(int(z["n_conv"])):
        c = orr.kl_curve(z[f"c{i}_masses"])
        np.testing.assert_allclose(c, z[f"c{i}_curve"], rtol=1e-12, atol=1e-15)
        curves.append(c)
    assert orr.detect_watershed(curves, "max_drop") == int(z["ws_max_drop_0.1"])
    assert orr.detect_watershed(curves, "threshold", 0.1) == int(z["ws_threshold_0.1"])
    assert orr.detect_watershed(curves, "threshold", 1e-3) == int(z["ws_threshold_0.001"])


def test_package_calibration_host_math_matches_reference():
    from paper_2502_15294_b200 import calibration as cal
    z = _calib()
    curves = [cal.kl_curve(z[f"c{i}_masses"]) for i in range(int(z["n_conv"]))]
    for i, c in enumerate(curves):
        np.testing.assert_allclose(c.values, z[f"c{i}_curve"], rtol=1e-12, atol=1e-15)
    assert cal.detect_watershed(curves).layer == int(z["ws_max_drop_0.1"])
    assert cal.detect_watershed(curves, "threshold", 1e-3).layer == int(z["ws_threshold_0.001"])
    assert cal.kl_divergence([0.5, 0.5], [0.5, 0.5]) == 0.0
    with pytest.raises(cal.DomainError):
        cal.detect_watershed(curves, "nope")


def test_package_memory_model_matches_reference():
    """The product package's Eq. 2 functions (paper_2502_15294_b200.store,
    store.py:308-357) against the reference's own outputs, bit-exact, plus the
    reference's validation errors."""
    from paper_2502_15294_b200 import store as pst
    from paper_2502_15294_b200.errors import DomainError
    data = load_store_cases()
    for m in data["memory"]:
        if "args" in m:
            L, lw, K, T = m["args"]
            assert pst.memory_ratio(L, lw, K, T) == float.fromhex(m["ratio"])
            assert pst.save_percent(L, lw) == m["save"]
            fp = pst.footprint_report(1, 1024, 4096, L, lw, K, T)
            for key, val in m["fp"].items():
                want = float.fromhex(val) if isinstance(val, str) else val
                assert fp[key] == want, (key, fp[key], want)
        else:
            L, lw = m["table5"]
            assert pst.save_percent(L, lw) == m["save"] == m["published"]
    assert pst.block_nbytes(1, 1920, 1) == 7680 and pst.block_nbytes(1, 3200, 1) == 12800
    for bad in ((4, 0, 1, 8), (4, 4, 1, 8), (4, 2, 9, 8), (4, 2, 1, 0)):
        with pytest.raises(DomainError):
            pst.memory_ratio(*bad)
    with pytest.raises(DomainError):
        pst.footprint_report(0, 1024, 4096, 32, 5, 4, 32)
