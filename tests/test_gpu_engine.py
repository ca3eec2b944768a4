"""GPU parity of the batched round-sparse serving engine (one full turn with
the model on the GPU): fused QKV projection + RoPE + KV append, decode
attention, output projection + residual per layer, the exact watershed scorer
and the device selector, the H2D gather of the kept rounds, the question's
upper layers and the greedy decode over the tied logits — against the oracle's
float64 restatement of the same turn (oracle/decode_model.py: the reference's
forward_range / run_turn, engine.py:244-271, pipeline.py:192-313, with the
engine's GQA shapes and bf16 weights / caches)."""

from __future__ import annotations

import dataclasses

import numpy as np
import pytest

from oracle import decode_model as odm
from oracle import rounds as orr

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2502_15294_b200 import kernels  # noqa: E402
from paper_2502_15294_b200.decode_engine import EngineConfig, GroupedDecoder, RoundDecodeEngine  # noqa: E402
from paper_2502_15294_b200.decode_model import DecodeModel  # noqa: E402
from paper_2502_15294_b200.selection import SelectionPolicy  # noqa: E402


def _f(t):
    return t.float().cpu().numpy()


def _oracle_turn(eng, model, b, lower0, variant=0, fraction=0.3):
    """The oracle's turn for dialogue b of `eng` (lower0: the lower caches before the turn)."""
    c = eng.cfg
    lw, T = c.watershed, c.round_tokens
    w = model.host_weights()
    orc = odm.TurnOracle(w, c.hq, c.hkv, c.head_dim, model.freq.cpu().numpy())
    hs = b % eng.host_sets

    def blocks(kept):
        out = []
        for u in range(eng.L_up):
            K = np.concatenate([_f(eng.host_blocks[hs][int(r)][u][0]) for r in kept])
            V = np.concatenate([_f(eng.host_blocks[hs][int(r)][u][1]) for r in kept])
            out.append((K, V))
        return out

    tok = int(eng.q_tok_all[variant, b, 0])
    return odm.run_turn(orc, [lower0[b, l, 0] for l in range(lw)], [lower0[b, l, 1] for l in range(lw)], blocks,
                        tok, eng.hist, T, c.rounds, lw, orr.SelectionPolicy("top_percent", fraction=fraction),
                        c.decode_steps)


def _small_cfg(**kw):
    base = dict(num_layers=4, watershed=2, hq=8, hkv=2, head_dim=128, rounds=7, round_tokens=64, batch=3,
                decode_steps=5, policy=SelectionPolicy("top_percent", fraction=0.3), item_chunk=32, plant=2,
                plant_beta=0.3, question_variants=1)
    base.update(kw)
    return EngineConfig(**base)


@pytest.mark.parametrize("graphs", [False, True])
@pytest.mark.parametrize("hkv,G", [(2, 4), (4, 7)])
def test_engine_turn_matches_oracle(graphs, hkv, G):
    cfg = _small_cfg(hq=hkv * G, hkv=hkv)
    model = DecodeModel(cfg.shape, "cuda", seed=3, prefill_gemm=True)
    eng = RoundDecodeEngine(cfg, model=model, dialogues=[5, 9, 13])
    lower0 = _f(eng.lower[:, :, :, : eng.hist])
    if graphs:
        eng.prepare()
        eng.slot_round[:] = -1
        kept, _ = eng.run_turn()
    else:
        with torch.cuda.stream(eng.compute_stream):
            kept = eng.run_turn_eager()
    torch.cuda.synchronize()
    answers = eng.answers()
    for b in range(cfg.batch):
        ref = _oracle_turn(eng, model, b, lower0)
        assert tuple(int(x) for x in kept[b]) == ref["kept"], b
        # the answer: SEP + greedy tokens; a flip would need a logit near-tie (gaps printed)
        assert list(answers[b]) == ref["answer"][:cfg.decode_steps], (b, list(answers[b]), ref["answer"],
                                                                      ref["logit_gaps"])
        assert int(eng.answer[b, cfg.decode_steps]) == ref["answer"][cfg.decode_steps]
        # after the last argmax the residual stream holds that token's embedding
        np.testing.assert_array_equal(_f(eng.x[b]), ref["x"])
    # the writeback holds this turn's upper rows
    wb = _f(eng.writeback)
    up = _f(eng.upper[:, :, :, eng.K * cfg.round_tokens: eng.K * cfg.round_tokens + eng.turn_rows])
    np.testing.assert_array_equal(wb, up)


def test_engine_hidden_states_match_oracle():
    """Hidden-state parity of the fused layer body (projections + RoPE +
    attention + residual): the question's rotated queries and residual stream
    after every lower layer within 1e-4 of the float64 oracle (fp32-class
    projections), and the appended key / value rows equal the oracle's bf16 rows."""
    cfg = _small_cfg(batch=2, decode_steps=2)
    model = DecodeModel(cfg.shape, "cuda", seed=11, prefill_gemm=True)
    eng = RoundDecodeEngine(cfg, model=model, dialogues=[0, 1])
    w = model.host_weights()
    orc = odm.TurnOracle(w, cfg.hq, cfg.hkv, cfg.head_dim, model.freq.cpu().numpy())
    lower0 = _f(eng.lower[:, :, :, : eng.hist])
    eng._set_question()
    eng._set_turn_lengths()
    eng.pos.copy_(eng.pos_q0)
    kernels.embed(eng.q_tok.view(-1), model.emb, eng.x)
    xs = [w["emb"][int(eng.q_tok[b, 0])].astype(np.float32) for b in range(2)]
    for b in range(2):
        np.testing.assert_array_equal(_f(eng.x[b]), xs[b])
    for l in range(cfg.watershed):
        eng._layer(l, advance=(l == cfg.watershed - 1))
        torch.cuda.synchronize()
        for b in range(2):
            xs[b], K, V, _, q = orc.layer(l, xs[b], eng.hist, lower0[b, l, 0], lower0[b, l, 1])
            np.testing.assert_allclose(_f(eng.q_buf[b]), q, rtol=1e-4, atol=1e-4)
            err = np.abs(_f(eng.x[b]) - xs[b]).max() / np.abs(xs[b]).max()
            assert err < 1e-4, (l, b, err)
            # appended rows: bf16 of fp32-class values; equal unless a value sits at a bf16 rounding boundary
            kd = np.abs(_f(eng.lower[b, l, 0, eng.hist]) - K[-1]).max()
            vd = np.abs(_f(eng.lower[b, l, 1, eng.hist]) - V[-1]).max()
            assert kd <= 1e-2 * np.abs(K[-1]).max() and vd <= 1e-2 * np.abs(V[-1]).max()


def test_engine_prefill_turn_matches_oracle():
    """Multi-row question (library-GEMM projections + RoPE rows, tcgen05 prefill
    attention with the Lw-1 scoring fused, fp64 re-score below the margin): the
    kept rounds equal the oracle's selection from the capture of ALL question
    rows (aggregate_round_attention over rows, stats.py:59-94)."""
    from oracle.attention import attention_forward_gqa, round_to_bf16
    nq = 40
    cfg = _small_cfg(round_tokens=128, batch=2, decode_steps=3, item_chunk=128, question_rows=nq)
    model = DecodeModel(cfg.shape, "cuda", seed=5, prefill_gemm=True)
    eng = RoundDecodeEngine(cfg, model=model, dialogues=[2, 3])
    c = cfg
    lw, T, R, hist = c.watershed, c.round_tokens, c.rounds, eng.hist
    lower0 = _f(eng.lower[:, :, :, :hist])
    with torch.cuda.stream(eng.compute_stream):
        kept = eng.run_turn_eager()
    torch.cuda.synchronize()
    w = model.host_weights()
    freq = model.freq.cpu().numpy()
    qpos = np.arange(hist, hist + nq)
    for b in range(c.batch):
        toks = [int(t) for t in eng.q_tok_all[0, b]]
        X = w["emb"][toks].astype(np.float64)                          # (nq, D)
        cap = None
        for l in range(lw):
            q = (X @ w["wq"][l]).astype(np.float32).reshape(nq, c.hq, c.head_dim)
            k = (X @ w["wk"][l]).astype(np.float32).reshape(nq, c.hkv, c.head_dim)
            v = (X @ w["wv"][l]).astype(np.float32).reshape(nq, c.hkv, c.head_dim)
            q = odm.rope(q, qpos, freq)
            k = round_to_bf16(odm.rope(k, qpos, freq))
            v = round_to_bf16(v)
            K = np.concatenate([lower0[b, l, 0], k])
            V = np.concatenate([lower0[b, l, 1], v])
            out, cp = attention_forward_gqa(q, K, V, qpos, np.arange(hist + nq), capture=(l == lw - 1))
            if l == lw - 1:
                cap = cp
            X = X + out.astype(np.float64) @ w["wo"][l]
        rounds = [orr.Round(r, (r * T, r * T + 1), (r * T + 1, (r + 1) * T)) for r in range(R)]
        rounds.append(orr.Round(R, (hist, hist + nq), (hist + nq, hist + nq)))
        raw = orr.aggregate_round_attention(cap, rounds, "question", R, row_offset=hist)
        want = orr.select(orr.normalize(raw), orr.SelectionPolicy("top_percent", fraction=0.3))
        assert tuple(int(x) for x in kept[b]) == want, b
        np.testing.assert_allclose(_f(eng.raw[b]), raw, rtol=1e-4, atol=1e-12)


def test_engine_prefill_graphs_match_eager():
    """Multi-row questions: the question's upper layers replayed as per-layer CUDA
    graphs (captured by prepare, replayed between the gather waits) give the eager
    turn's kept rounds, raw masses and answer ids bit for bit, over turns whose
    questions, kept rounds and working-cache slot positions change."""
    nq = 24
    cfg = _small_cfg(round_tokens=128, batch=2, decode_steps=4, item_chunk=128, question_rows=nq,
                     question_variants=3)
    model = DecodeModel(cfg.shape, "cuda", seed=9, prefill_gemm=True)
    ref = RoundDecodeEngine(cfg, model=model, dialogues=[4, 5])
    eng = RoundDecodeEngine(cfg, model=model, dialogues=[4, 5])
    eng.prepare()                    # one eager warm-up turn, then the graphs
    assert eng.graphs_b1 is not None and len(eng.graphs_b1) == cfg.num_layers - cfg.watershed
    with torch.cuda.stream(ref.compute_stream):
        ref.run_turn_eager()         # the same warm-up turn on the eager engine
    for _ in range(3):
        with torch.cuda.stream(ref.compute_stream):
            kr = ref.run_turn_eager()
        kg, _ = eng.run_turn()
        torch.cuda.synchronize()
        assert [list(map(int, k)) for k in kr] == [list(map(int, k)) for k in kg]
        assert torch.equal(ref.raw, eng.raw)
        np.testing.assert_array_equal(ref.answers(), eng.answers())


def test_engine_e2e_matches_device_path():
    """The public-API turn (question ids from pinned host memory, answer ids
    back to it) gives the device-resident turn's kept rounds and answers."""
    cfg = _small_cfg(rounds=6, batch=2, decode_steps=9, plant=1)
    eng = RoundDecodeEngine(cfg, dialogues=[0, 1])
    eng.prepare(e2e=True)
    kept, _ = eng.run_turn(e2e=False)
    torch.cuda.synchronize()
    ans = eng.answer.cpu().clone()
    kept_e, _ = eng.run_turn(e2e=True)
    eng.compute_stream.synchronize()
    torch.cuda.synchronize()
    assert [list(map(int, k)) for k in kept] == [list(map(int, k)) for k in kept_e]
    assert torch.equal(eng.answer_host, ans)


def test_engine_round_cache_reuses_slots():
    """Cross-turn round cache: a round kept again stays in its working-cache
    slot (no H2D); with the same question every turn nothing is re-fetched and
    the answers are identical to the first turn's; with varying questions only
    the newly kept rounds are fetched."""
    eng = RoundDecodeEngine(_small_cfg(rounds=8, batch=2, decode_steps=3), dialogues=[21, 22])
    eng.prepare()
    eng.slot_round[:] = -1                     # cold cache
    _, b0 = eng.run_turn()
    torch.cuda.synchronize()
    ans0 = eng.answer.clone()
    assert eng.last_copied_rounds == 2 * eng.K and b0 > 0
    _, b1 = eng.run_turn()
    torch.cuda.synchronize()
    assert eng.last_copied_rounds == 0 and b1 == 0
    assert torch.equal(eng.answer, ans0)
    eng2 = RoundDecodeEngine(_small_cfg(rounds=8, batch=2, decode_steps=3, question_variants=3), dialogues=[21, 22])
    eng2.prepare()
    prev = None
    for _ in range(4):
        kept, _ = eng2.run_turn()
        torch.cuda.synchronize()
        now = [set(int(x) for x in k) for k in kept]
        if prev is not None:
            assert eng2.last_copied_rounds == sum(len(n - p) for n, p in zip(now, prev))
        for b in range(2):
            assert set(int(x) for x in eng2.slot_round[b]) == now[b]
        prev = now


@pytest.mark.parametrize("stagger", [True, False])
def test_grouped_decoder_matches_single_engine(stagger):
    """The bench's serving shape: two dialogue groups on their own streams
    sharing one model, the second starting after the first group's first KV
    gather (stagger) or both at once (their scoring and selection overlap on
    the device: each engine owns its workspaces).  Kept rounds and answers
    equal standalone engines' eager turns bit for bit; e2e path."""
    cfg = _small_cfg(batch=4, decode_steps=5, plant=0)
    gd = GroupedDecoder(cfg, groups=2, dialogues=[10, 11, 12, 13])
    gd.stagger = stagger
    assert gd.groups[0].ws.data_ptr() != gd.groups[1].ws.data_ptr()
    assert gd.groups[0].ws_exact.data_ptr() != gd.groups[1].ws_exact.data_ptr()
    gd.prepare(e2e=True)
    gd.run_turns(3, e2e=True)
    torch.cuda.synchronize()
    sub = dataclasses.replace(cfg, batch=2)
    for g, eng in enumerate(gd.groups):
        ref = RoundDecodeEngine(sub, model=gd.model, dialogues=[10 + 2 * g, 11 + 2 * g])
        with torch.cuda.stream(ref.compute_stream):
            kept = ref.run_turn_eager()
        torch.cuda.synchronize()
        assert [tuple(int(x) for x in k) for k in kept] == [tuple(int(x) for x in k) for k in eng.last_kept]
        assert torch.equal(eng.answer_host, ref.answer.cpu())


def test_sharding_invariance_kept_and_answers():
    """Dialogues are data-seeded by their global id: the same dialogues served
    as one batch or split across two engines (two ranks' shards, b mod 2) give
    identical kept rounds and answers (multi-GPU weak scaling)."""
    cfg = _small_cfg(batch=4, decode_steps=4, question_variants=2)
    model = DecodeModel(cfg.shape, "cuda", seed=42)
    whole = RoundDecodeEngine(cfg, model=model, dialogues=[0, 1, 2, 3])
    with torch.cuda.stream(whole.compute_stream):
        k_all = whole.run_turn_eager()
    torch.cuda.synchronize()
    half = dataclasses.replace(cfg, batch=2)
    for r in range(2):
        shard = RoundDecodeEngine(half, model=model, dialogues=[r, r + 2])
        with torch.cuda.stream(shard.compute_stream):
            k_sh = shard.run_turn_eager()
        torch.cuda.synchronize()
        for i, gid in enumerate([r, r + 2]):
            assert tuple(map(int, k_sh[i])) == tuple(map(int, k_all[gid]))
            assert torch.equal(shard.answer[i].cpu(), whole.answer[gid].cpu())


def test_engine_accounting():
    cfg = EngineConfig(num_layers=32, watershed=5, hq=32, hkv=8, head_dim=128, rounds=32, round_tokens=512, batch=1,
                       decode_steps=2, plant=0)
    eng = RoundDecodeEngine(cfg)
    resident, full = eng.gpu_kv_bytes()
    assert 1 - resident / full > 0.54                      # >= 54 % GPU KV saved (north star)
    assert eng.K == 4
    # Llama-3-8B-shaped projections: 41.9 M parameters per layer (bf16), + the tied logits (vocab 258)
    per_layer = (4096 * (32 + 16) * 128 + 4096 * 4096) * 2
    assert eng.weight_bytes_per_token() == 32 * per_layer + 4096 * 258 * 2


def test_engine_c2_full_shapes_turn_matches_oracle():
    """One graph-replayed turn at the bench's C2 shapes (32 layers, Lw=5, 32
    heads over 8 kv-heads, 32 rounds x 512 keys, K=4; two dialogues): the kept
    rounds and the answer ids equal the float64 oracle's turn."""
    cfg = EngineConfig(num_layers=32, watershed=5, hq=32, hkv=8, head_dim=128, rounds=32, round_tokens=512,
                       batch=2, decode_steps=3, policy=SelectionPolicy("top_percent", fraction=0.10), plant=2,
                       plant_beta=0.25, question_variants=1)
    model = DecodeModel(cfg.shape, "cuda", seed=42, prefill_gemm=True)
    eng = RoundDecodeEngine(cfg, model=model, dialogues=[0, 1])
    lower0 = _f(eng.lower[:, :, :, : eng.hist])
    eng.prepare()
    eng.slot_round[:] = -1
    kept, _ = eng.run_turn()
    torch.cuda.synchronize()
    answers = eng.answers()
    for b in range(cfg.batch):
        ref = _oracle_turn(eng, model, b, lower0, fraction=0.10)
        assert tuple(int(x) for x in kept[b]) == ref["kept"]
        assert list(answers[b]) == ref["answer"][:cfg.decode_steps], ref["logit_gaps"]
