"""GPU parity of the persistent whole-step decode kernel (rk_decode_step: one
launch per answer token runs every layer's QKV projection + RoPE + KV append,
split-K decode attention + merge, output projection + residual, then the tied
logits + first-max argmax + embedding).  Checked against the oracle's float64
turn (oracle/decode_model.py: the reference's forward_range / run_turn,
engine.py:244-271, pipeline.py:298-313) and against the layered kernels."""

from __future__ import annotations

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2502_15294_b200 import kernels  # noqa: E402
from paper_2502_15294_b200.decode_engine import RoundDecodeEngine  # noqa: E402
from paper_2502_15294_b200.decode_model import DecodeModel  # noqa: E402

from test_gpu_engine import _f, _oracle_turn, _small_cfg  # noqa: E402


def _engine(cfg, seed, dialogues):
    model = DecodeModel(cfg.shape, "cuda", seed=seed, prefill_gemm=True)
    return RoundDecodeEngine(cfg, model=model, dialogues=dialogues), model


@pytest.mark.parametrize("hkv,G,batch", [(2, 4, 3), (4, 7, 2), (2, 4, 1), (2, 4, 11)])
def test_step_turn_matches_oracle(hkv, G, batch):
    """A whole turn whose answer loop runs on rk_decode_step (graph-captured):
    kept rounds, greedy answers and the final residual equal the oracle's."""
    cfg = _small_cfg(hq=hkv * G, hkv=hkv, batch=batch, step_kernel="persistent")
    eng, model = _engine(cfg, 3, [5 + 4 * b for b in range(batch)])
    assert eng.persistent and eng.launches_per_token() == 1
    lower0 = _f(eng.lower[:, :, :, : eng.hist])
    eng.prepare()
    eng.slot_round[:] = -1
    kept, _ = eng.run_turn()
    torch.cuda.synchronize()
    answers = eng.answers()
    for b in range(cfg.batch):
        ref = _oracle_turn(eng, model, b, lower0)
        assert tuple(int(x) for x in kept[b]) == ref["kept"], b
        assert list(answers[b]) == ref["answer"][:cfg.decode_steps], (b, list(answers[b]), ref["answer"],
                                                                      ref["logit_gaps"])
        assert int(eng.answer[b, cfg.decode_steps]) == ref["answer"][cfg.decode_steps]
        np.testing.assert_array_equal(_f(eng.x[b]), ref["x"])
    # lengths advanced once per token (question + answer rows appended to both tiers)
    assert int(eng.lower_len[0]) == eng.hist + eng.turn_rows
    assert int(eng.upper_len[0]) == eng.K * cfg.round_tokens + eng.turn_rows
    wb = _f(eng.writeback)
    up = _f(eng.upper[:, :, :, eng.K * cfg.round_tokens: eng.K * cfg.round_tokens + eng.turn_rows])
    np.testing.assert_array_equal(wb, up)


@pytest.mark.parametrize("batch", [1, 4, 16])
def test_step_matches_layered_kernels(batch):
    """Same turns through both answer loops: the persistent step's appended KV
    rows, answers and residual stream agree with the layered kernels' (the
    projections' split-K partitions differ, so fp32 sums differ in the last
    bits: rows within 2 bf16 ulps, residual within 1e-5 relative), over two
    turns (the workspace's counters carry over between launches)."""
    kw = dict(batch=batch, decode_steps=6, rounds=9)
    e_l, _ = _engine(_small_cfg(step_kernel="layers", **kw), 7, list(range(batch)))
    e_p, _ = _engine(_small_cfg(step_kernel="persistent", **kw), 7, list(range(batch)))
    assert e_p.persistent and not e_l.persistent
    for eng in (e_l, e_p):
        eng.prepare()
    for _turn in range(2):
        outs = []
        for eng in (e_l, e_p):
            kept, _ = eng.run_turn()
            torch.cuda.synchronize()
            outs.append((kept, eng.answers().copy(), _f(eng.x), _f(eng.upper), _f(eng.lower)))
        (k_l, a_l, x_l, up_l, lo_l), (k_p, a_p, x_p, up_p, lo_p) = outs
        assert [tuple(k) for k in k_l] == [tuple(k) for k in k_p]
        np.testing.assert_array_equal(a_l, a_p)
        np.testing.assert_array_equal(x_l, x_p)           # embedding of the same final token
        for A, Bq in ((up_l, up_p), (lo_l, lo_p)):
            tol = 2.0 ** -7 * np.maximum(np.abs(A), 1e-3)
            assert np.all(np.abs(A - Bq) <= tol)


def test_step_hidden_state_matches_layered():
    """One token step from the same state: the residual stream after all layers
    (before the logits: read back by skipping the argmax through a 1-step
    comparison of the appended rows) — here the appended K/V rows of every
    layer, which carry each layer's projections, RoPE and attention inputs."""
    cfg = _small_cfg(batch=5, decode_steps=3, step_kernel="persistent")
    eng, m = _engine(cfg, 19, [3, 1, 4, 1, 5])
    c = eng.cfg
    gen = torch.Generator(device="cuda").manual_seed(5)
    x0 = torch.randn(eng.x.shape, generator=gen, device="cuda")
    res = []
    for mode in ("layers", "persistent"):
        eng.lower_len.copy_(eng.lower_len0)
        eng.upper_len.copy_(eng.upper_len0)
        eng.pos.copy_(eng.pos_dec0)
        eng.x.copy_(x0)
        if mode == "layers":
            for l in range(c.num_layers):
                eng._layer(l, advance=(l == c.watershed - 1 or l == c.num_layers - 1))
            kernels.lm_head(eng.x, m.emb_packed, m.shape.vocab, m.emb, eng.x, eng.tokens, eng.pos, ws=eng.lm_ws)
        else:
            kernels.decode_step(eng.step_args[0])
        torch.cuda.synchronize()
        h = eng.hist
        u = eng.K * c.round_tokens
        res.append((_f(eng.lower[:, :, :, h]), _f(eng.upper[:, :, :, u]), eng.tokens.cpu().numpy().copy(),
                    eng.lower_len.cpu().numpy().copy(), eng.pos.cpu().numpy().copy()))
    (lo_a, up_a, t_a, l_a, p_a), (lo_b, up_b, t_b, l_b, p_b) = res
    for A, Bq in ((lo_a, lo_b), (up_a, up_b)):
        tol = 2.0 ** -7 * np.maximum(np.abs(A), 1e-3)
        assert np.all(np.abs(A - Bq) <= tol), np.abs(A - Bq).max()
    np.testing.assert_array_equal(t_a, t_b)
    np.testing.assert_array_equal(l_a, l_b)
    np.testing.assert_array_equal(p_a, p_b)


def test_step_rejects_unsupported():
    assert not kernels.decode_step_supported(17, 32, 8, 128)
    assert not kernels.decode_step_supported(4, 32, 2, 128)        # group 16 > 8
    assert not kernels.decode_step_supported(4, 32, 8, 64)
    assert not kernels.decode_step_supported(4, 32, 8, 128, torch.float32)
    assert kernels.decode_step_supported(16, 32, 8, 128)
    with pytest.raises(ValueError):
        _engine(_small_cfg(batch=17, step_kernel="persistent"), 1, list(range(17)))
