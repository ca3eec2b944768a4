"""GPU parity of the batched round-sparse decode engine (one full turn):
fused watershed scoring + device selection must pick the oracle's rounds
bit-exactly, the H2D gather must assemble exactly the kept rounds' deep-layer
KV, and the decode outputs after T tokens must match the oracle attention over
(kept rounds + this turn's tokens) in the upper layers and the full history in
the lower layers (pipeline.py:192-394 semantics)."""

from __future__ import annotations

import numpy as np
import pytest

from oracle import attention as oatt
from oracle import rounds as orr

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2502_15294_b200.decode_engine import EngineConfig, RoundDecodeEngine  # noqa: E402
from paper_2502_15294_b200.selection import SelectionPolicy  # noqa: E402


def _f(t):
    return t.float().cpu().numpy()


@pytest.mark.parametrize("graphs", [False, True])
@pytest.mark.parametrize("hkv,G", [(2, 4), (4, 7)])
def test_engine_turn_matches_oracle(graphs, hkv, G):
    cfg = EngineConfig(num_layers=4, watershed=2, hq=hkv * G, hkv=hkv, head_dim=128, rounds=7, round_tokens=64,
                       batch=3, decode_steps=5, policy=SelectionPolicy("top_percent", fraction=0.3),
                       item_chunk=32, input_period=3, plant=2, plant_beta=0.3)
    eng = RoundDecodeEngine(cfg, seed=3)
    lw, L, T, R = cfg.watershed, cfg.num_layers, cfg.round_tokens, cfg.rounds
    lower0 = _f(eng.lower[:, :, :, : eng.hist])          # history before the turn
    if graphs:
        eng.prepare(e2e=False)
        kept, _ = eng.run_turn()
        kept, _ = eng.run_turn()                          # steady state: second replay
    else:
        with torch.cuda.stream(eng.compute_stream):
            kept = eng.run_turn_eager()
    torch.cuda.synchronize()
    P = eng.period
    steps = eng.turn_tokens
    for b in range(cfg.batch):
        # ---- selection: oracle capture at layer Lw-1 for the question token
        q0 = _f(eng.q_in[0, lw - 1, b])[None]
        kq = np.concatenate([lower0[b, lw - 1, 0], _f(eng.kv_in[0, lw - 1, 0, b])[None]])
        _, cap = oatt.attention_forward_gqa(q0, kq, kq, [eng.hist], np.arange(eng.hist + 1), capture=True)
        raw = np.array([cap[0, r * T:(r + 1) * T].sum() for r in range(R)])
        want = orr.select(orr.normalize(raw), orr.SelectionPolicy("top_percent", fraction=0.3))
        assert tuple(int(x) for x in kept[b]) == want
        assert set(eng.planted[b]) <= set(want)
        # ---- last token: lower layer 0 over history + the turn's rows, upper layer L-1 over kept + rows
        tl = steps - 1
        for l in (0, lw - 1, lw, L - 1):
            rows_k = np.stack([_f(eng.kv_in[t % P, l, 0, b]) for t in range(steps)])
            rows_v = np.stack([_f(eng.kv_in[t % P, l, 1, b]) for t in range(steps)])
            if l < lw:
                K = np.concatenate([lower0[b, l, 0], rows_k])
                V = np.concatenate([lower0[b, l, 1], rows_v])
            else:
                hs = b % eng.host_sets
                blocks = [eng.host_blocks[hs][int(r)][l - lw] for r in kept[b]]
                K = np.concatenate([_f(bk[0]) for bk in blocks] + [rows_k])
                V = np.concatenate([_f(bk[1]) for bk in blocks] + [rows_v])
            q = _f(eng.q_in[tl % P, l, b])[None]
            ref, _ = oatt.attention_forward_gqa(q, K, V, [len(K) - 1], np.arange(len(K)))
            got = _f(eng.out[l, b]).reshape(1, -1)
            err = np.abs(got - ref).max() / np.abs(ref).max()
            assert err < 1e-4, (l, err)
        # ---- writeback holds this turn's upper rows
        wb = _f(eng.writeback[b])
        up = _f(eng.upper[b, :, :, eng.K * T: eng.K * T + steps])
        np.testing.assert_array_equal(wb, up)


def test_engine_accounting():
    cfg = EngineConfig(num_layers=32, watershed=5, hq=32, hkv=8, head_dim=128, rounds=32, round_tokens=512, batch=1,
                       decode_steps=2, plant=0)
    eng = RoundDecodeEngine(cfg)
    resident, full = eng.gpu_kv_bytes()
    assert 1 - resident / full > 0.54                      # >= 54 % GPU KV saved (north star)
    assert eng.K == 4


@pytest.mark.parametrize("graphs", [False, True])
def test_engine_prefill_turn_matches_oracle(graphs):
    """Multi-row question (tcgen05 prefill, fused scoring at Lw-1): kept rounds
    equal the oracle's selection from the capture of ALL question rows
    (aggregate_round_attention over rows, stats.py:59-94); the question's upper
    layers attend kept rounds + the question with original positions
    (pipeline.py:292-296); the decode tokens then see the history / kept
    rounds plus every row of the turn."""
    nq, hkv, G = 40, 2, 4
    cfg = EngineConfig(num_layers=4, watershed=2, hq=hkv * G, hkv=hkv, head_dim=128, rounds=7, round_tokens=128,
                       batch=2, decode_steps=4, policy=SelectionPolicy("top_percent", fraction=0.3),
                       item_chunk=128, input_period=3, plant=2, plant_beta=0.3, question_rows=nq)
    eng = RoundDecodeEngine(cfg, seed=5)
    lw, L, T, R, hist = cfg.watershed, cfg.num_layers, cfg.round_tokens, cfg.rounds, eng.hist
    lower0 = _f(eng.lower[:, :, :, :hist])
    if graphs:
        eng.prepare(e2e=False)
        kept, _ = eng.run_turn()
        kept, _ = eng.run_turn()
    else:
        with torch.cuda.stream(eng.compute_stream):
            kept = eng.run_turn_eager()
    torch.cuda.synchronize()
    P = eng.period
    qpos = np.arange(hist, hist + nq)
    for b in range(cfg.batch):
        # ---- selection from the question rows' capture at layer Lw-1
        qq = _f(eng.qq_in[lw - 1, b])
        kq = np.concatenate([lower0[b, lw - 1, 0], _f(eng.qkv_in[lw - 1, 0, b])])
        _, cap = oatt.attention_forward_gqa(qq, kq, kq, qpos, np.arange(hist + nq), capture=True)
        rounds = [orr.Round(r, (r * T, r * T + 1), (r * T + 1, (r + 1) * T)) for r in range(R)]
        rounds.append(orr.Round(R, (hist, hist + nq), (hist + nq, hist + nq)))
        raw = orr.aggregate_round_attention(cap, rounds, "question", R, active_rounds=list(range(R)),
                                            row_offset=hist)
        want = orr.select(orr.normalize(raw), orr.SelectionPolicy("top_percent", fraction=0.3))
        assert tuple(int(x) for x in kept[b]) == want
        # ---- last decode token at a lower and an upper layer
        for l in (0, lw - 1, lw, L - 1):
            qk, qv = _f(eng.qkv_in[l, 0, b]), _f(eng.qkv_in[l, 1, b])
            rows_k = np.stack([_f(eng.kv_in[t % P, l, 0, b]) for t in range(1, cfg.decode_steps + 1)])
            rows_v = np.stack([_f(eng.kv_in[t % P, l, 1, b]) for t in range(1, cfg.decode_steps + 1)])
            if l < lw:
                K = np.concatenate([lower0[b, l, 0], qk, rows_k])
                V = np.concatenate([lower0[b, l, 1], qv, rows_v])
            else:
                hs = b % eng.host_sets
                blocks = [eng.host_blocks[hs][int(r)][l - lw] for r in kept[b]]
                K = np.concatenate([_f(bk[0]) for bk in blocks] + [qk, rows_k])
                V = np.concatenate([_f(bk[1]) for bk in blocks] + [qv, rows_v])
            q = _f(eng.q_in[cfg.decode_steps % P, l, b])[None]
            ref, _ = oatt.attention_forward_gqa(q, K, V, [len(K) - 1], np.arange(len(K)))
            err = np.abs(_f(eng.out[l, b]).reshape(1, -1) - ref).max() / np.abs(ref).max()
            assert err < 1e-4, (l, err)
        # ---- the question's last upper layer: kept rounds + causal question, original positions
        blocks = [eng.host_blocks[b % eng.host_sets][int(r)][L - 1 - lw] for r in kept[b]]
        K = np.concatenate([_f(bk[0]) for bk in blocks] + [_f(eng.qkv_in[L - 1, 0, b])])
        V = np.concatenate([_f(bk[1]) for bk in blocks] + [_f(eng.qkv_in[L - 1, 1, b])])
        kpos = np.concatenate([np.arange(int(r) * T, (int(r) + 1) * T) for r in kept[b]] + [qpos])
        ref, _ = oatt.attention_forward_gqa(_f(eng.qq_in[L - 1, b]), K, V, qpos, kpos)
        got = _f(eng.qout[b]).reshape(nq, -1)
        assert np.abs(got - ref).max() / np.abs(ref).max() < 1e-4


def test_engine_e2e_pipeline_matches_device_path():
    """End-to-end turn (inputs from pinned host memory, outputs back to it, the
    copies pipelined on a side stream against the decode kernels) produces
    exactly the device-resident turn's outputs for every token."""
    cfg = EngineConfig(num_layers=4, watershed=2, hq=16, hkv=4, head_dim=128, rounds=6, round_tokens=64, batch=2,
                       decode_steps=9, policy=SelectionPolicy("top_percent", fraction=0.3), item_chunk=32,
                       input_period=3, plant=1, question_variants=1)     # identical turns
    eng = RoundDecodeEngine(cfg, seed=11)
    eng.prepare(e2e=True)
    T = cfg.decode_steps
    want = []
    for _ in range(2):
        eng.run_turn(e2e=False)
        torch.cuda.synchronize()
    # device path, token by token: replay the answer phase eagerly to collect every token's outputs
    kept, _ = eng.run_turn(e2e=False)
    torch.cuda.synchronize()
    last_dev = eng.out.clone()
    kept_e, _ = eng.run_turn(e2e=True)
    eng.compute_stream.synchronize()
    torch.cuda.synchronize()
    assert [list(map(int, k)) for k in kept] == [list(map(int, k)) for k in kept_e]
    assert torch.equal(eng.host_out[T], last_dev.cpu())
    assert torch.equal(eng.host_out[T], eng.out_buf[T % 2].cpu())
    want = eng.host_out[1:T + 1].clone()
    eng.run_turn(e2e=True)
    torch.cuda.synchronize()
    assert torch.equal(eng.host_out[1:T + 1], want)      # every token, turn after turn


def test_engine_round_cache_reuses_slots():
    """Cross-turn round cache: a round kept again stays in its working-cache
    slot (no H2D); with the same question every turn nothing is re-fetched and
    the outputs are bit-identical to the first turn's; with varying questions
    only the newly kept rounds are fetched and outputs still match the oracle
    (checked by test_engine_turn_matches_oracle)."""
    base = dict(num_layers=4, watershed=2, hq=16, hkv=4, head_dim=128, rounds=8, round_tokens=64, batch=2,
                decode_steps=3, policy=SelectionPolicy("top_percent", fraction=0.3), item_chunk=32, plant=2)
    eng = RoundDecodeEngine(EngineConfig(**base, question_variants=1), seed=21)
    eng.prepare()                              # (its warm-up turn already fills the slots)
    eng.slot_round[:] = -1                     # cold cache
    _, b0 = eng.run_turn()
    torch.cuda.synchronize()
    out0 = eng.out.clone()
    assert eng.last_copied_rounds == 2 * eng.K and b0 > 0
    kept, b1 = eng.run_turn()
    torch.cuda.synchronize()
    assert eng.last_copied_rounds == 0 and b1 == 0
    assert torch.equal(eng.out, out0)
    # varying questions: only rounds not already resident are fetched
    eng2 = RoundDecodeEngine(EngineConfig(**base, question_variants=3, question_noise=1.0), seed=21)
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
def test_grouped_decoder_e2e_matches_single_engine(stagger):
    """The bench's serving shape: two dialogue groups on their own streams, the
    second starting after the first group's first KV gather (stagger) or both at
    once (their scoring layers and selections overlap on the device: each engine
    must own its decode workspace), every token's activations loaded from pinned
    host memory and outputs read back (e2e).  Kept rounds and the last token's
    outputs equal a standalone engine's eager turn bit for bit."""
    import dataclasses

    from paper_2502_15294_b200.decode_engine import GroupedDecoder
    cfg = EngineConfig(num_layers=4, watershed=2, hq=8, hkv=2, head_dim=128, rounds=7, round_tokens=64,
                       batch=4, decode_steps=5, policy=SelectionPolicy("top_percent", fraction=0.3),
                       item_chunk=32, input_period=3, plant=0, question_variants=1)
    gd = GroupedDecoder(cfg, groups=2, seed=11)
    gd.stagger = stagger
    assert gd.groups[0].ws.data_ptr() != gd.groups[1].ws.data_ptr()
    gd.prepare(e2e=True)
    gd.run_turns(3, e2e=True)
    torch.cuda.synchronize()
    sub = dataclasses.replace(cfg, batch=2)
    for g, eng in enumerate(gd.groups):
        ref = RoundDecodeEngine(sub, seed=11 + 97 * g)
        with torch.cuda.stream(ref.compute_stream):
            kept = ref.run_turn_eager()
        torch.cuda.synchronize()
        assert [tuple(int(x) for x in k) for k in kept] == [tuple(int(x) for x in k) for k in eng.last_kept]
        T = cfg.decode_steps
        assert torch.equal(eng.host_out[T], ref.out.cpu())


def test_engine_c2_full_shapes_turn_matches_oracle():
    """One graph-replayed turn at the bench's C2 shapes (32 layers, Lw=5, 32 heads
    over 8 kv-heads, 32 rounds x 512 keys, K=4; two dialogues): the kept rounds
    equal the oracle's selection from the capture at layer Lw-1 over all 16 K
    history keys, and the last token's outputs at layers 0, Lw-1, Lw, L-1 equal the
    oracle over the full history / the kept rounds plus the turn's rows."""
    cfg = EngineConfig(num_layers=32, watershed=5, hq=32, hkv=8, head_dim=128, rounds=32, round_tokens=512,
                       batch=2, decode_steps=3, policy=SelectionPolicy("top_percent", fraction=0.10),
                       input_period=3, plant=2, plant_beta=0.25, question_variants=1)
    eng = RoundDecodeEngine(cfg, seed=5)
    lw, L, T, R = cfg.watershed, cfg.num_layers, cfg.round_tokens, cfg.rounds
    lower0 = {(b, l): (_f(eng.lower[b, l, 0, : eng.hist]), _f(eng.lower[b, l, 1, : eng.hist]))
              for b in range(cfg.batch) for l in (0, lw - 1)}
    eng.prepare(e2e=False)
    kept, _ = eng.run_turn()
    torch.cuda.synchronize()
    P, steps = eng.period, eng.turn_tokens
    assert eng.K == 4
    for b in range(cfg.batch):
        q0 = _f(eng.q_in[0, lw - 1, b])[None]
        kq = np.concatenate([lower0[(b, lw - 1)][0], _f(eng.kv_in[0, lw - 1, 0, b])[None]])
        _, cap = oatt.attention_forward_gqa(q0, kq, kq, [eng.hist], np.arange(eng.hist + 1), capture=True)
        raw = np.array([cap[0, r * T:(r + 1) * T].sum() for r in range(R)])
        want = orr.select(orr.normalize(raw), orr.SelectionPolicy("top_percent", fraction=0.10))
        assert tuple(int(x) for x in kept[b]) == want
        tl = steps - 1
        for l in (0, lw - 1, lw, L - 1):
            rows_k = np.stack([_f(eng.kv_in[t % P, l, 0, b]) for t in range(steps)])
            rows_v = np.stack([_f(eng.kv_in[t % P, l, 1, b]) for t in range(steps)])
            if l < lw:
                K = np.concatenate([lower0[(b, l)][0], rows_k])
                V = np.concatenate([lower0[(b, l)][1], rows_v])
            else:
                hs = b % eng.host_sets
                blocks = [eng.host_blocks[hs][int(r)][l - lw] for r in kept[b]]
                K = np.concatenate([_f(bk[0]) for bk in blocks] + [rows_k])
                V = np.concatenate([_f(bk[1]) for bk in blocks] + [rows_v])
            q = _f(eng.q_in[tl % P, l, b])[None]
            ref, _ = oatt.attention_forward_gqa(q, K, V, [len(K) - 1], np.arange(len(K)))
            got = _f(eng.out[l, b]).reshape(1, -1)
            err = np.abs(got - ref).max() / np.abs(ref).max()
            assert err < 1e-4, (b, l, err)
