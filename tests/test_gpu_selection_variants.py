"""SURVEY §8d's synthetic variants at C2 shapes (32 rounds x 512 keys, Hkv=8,
G=4, d=128; one decode token per dialogue): the fused watershed scoring of the
decode kernel (round items at layer Lw-1, pipeline.py:225-245 ->
stats.py:59-94) followed by the batched selector (selection.py:87-97), against
the oracle's capture + aggregate + normalize + select:
  * unplanted keys (hard parity: the K-boundary gap is small) — kept sets equal
    wherever the oracle's gap exceeds the masses' tolerance; the minimum gap
    seen is reported;
  * exact ties (duplicated rounds straddling the K boundary) — the masses of
    identical rounds must be bit-identical so ties go to the lower index, as
    the reference's stable argsort does;
  * zero mass (every round inactive) — the degenerate distribution."""

from __future__ import annotations

import numpy as np
import pytest

from oracle import attention as oatt
from oracle import rounds as orr

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2502_15294_b200 import kernels  # noqa: E402

R, T, HKV, G, D = 32, 512, 8, 4, 128
S = R * T
K = orr.top_k_count(R, 0.10, 1)           # 4


def _dialogues(B, seed, plant=None):
    """K/V caches [B][S+1][Hkv][d] bf16 and q [B][Hq][d]; plant(b, k, qn) edits k."""
    rng = np.random.default_rng(seed)
    q = rng.standard_normal((B, HKV * G, D)).astype(np.float32)
    k = rng.standard_normal((B, S + 1, HKV, D)).astype(np.float32)
    v = rng.standard_normal((B, S + 1, HKV, D)).astype(np.float32)
    if plant:
        for b in range(B):
            u = q[b].reshape(HKV, G, D).mean(axis=1)
            u /= np.linalg.norm(u, axis=-1, keepdims=True)
            plant(b, k[b], u)
    return q, oatt.round_to_bf16(k), oatt.round_to_bf16(v)


def _gpu_scores(q, k, v, active=None):
    B = q.shape[0]
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()  # noqa: E731
    kc, vc, tq = t(k).bfloat16(), t(v).bfloat16(), t(q)
    # the appended (current) row is the cache's last row; seq_len counts the history
    kn, vn = kc[:, S].clone(), vc[:, S].clone()
    sl = torch.full((B,), S, dtype=torch.int32, device="cuda")
    bounds = [[(m * T, (m + 1) * T, m) for m in range(R)] + [(S, S + 1, R)]] * B
    items, n_items = kernels.items_tensor(bounds, 256, "cuda")
    ws = kernels.decode_workspace(B, HKV * G, HKV, D, items.shape[1], "cuda", tag="sel_variants")
    kernels.decode_attention(tq, kc, vc, sl, S + 1, k_new=kn, v_new=vn, items=items, n_items=n_items, ws=ws)
    act = None if active is None else torch.from_numpy(active.astype(np.uint8)).cuda()
    raw = kernels.decode_scores_finalize(B, HKV * G, HKV, D, items, n_items, R, ws, active=act,
                                         kv_dtype=torch.bfloat16)
    masses, kept, meta = kernels.select_batch(raw, "top_percent", k_top=K)
    torch.cuda.synchronize()
    n_kept = meta[0].cpu().numpy()
    kept_sets = [tuple(sorted(int(x) for x in kept[b, :n_kept[b]].cpu().numpy())) for b in range(B)]
    return raw.cpu().numpy(), kept_sets, meta.cpu().numpy()


def _oracle(q, k, v, b, active=None):
    ref_out, cap = oatt.attention_forward_gqa(q[b:b + 1], k[b], v[b], [S], np.arange(S + 1), capture=True)
    act = np.ones(R, bool) if active is None else active
    raw = np.array([cap[0, m * T:(m + 1) * T].sum() if act[m] else 0.0 for m in range(R)])
    dist = orr.normalize(raw)
    kept = orr.select(dist, orr.SelectionPolicy("top_percent", fraction=0.10))
    return raw, tuple(kept), dist


def test_unplanted_hard_parity():
    """The fused fp32-class scoring's margin contract, with no tolerance escape:
    where its K-boundary margin clears the engines' refinement threshold (1e-3)
    its kept set IS the reference's; below it the engines re-score with the
    exact fp64 scorer, whose kept set is the reference's too."""
    B = 8
    q, k, v = _dialogues(B, seed=2002)
    raw, kept, _ = _gpu_scores(q, k, v)
    masses = torch.from_numpy(raw / raw.sum(axis=1, keepdims=True)).cuda()
    margin = kernels.selection_margin(masses, "top_percent", k_top=K).cpu().numpy()
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()  # noqa: E731
    bounds = [[(m * T, (m + 1) * T, m) for m in range(R)] + [(S, S + 1, R)]] * B
    items, n_items = kernels.items_tensor(bounds, 1024, "cuda")
    raw_ex = kernels.round_scores_exact(t(q)[:, None], t(k).bfloat16(), torch.tensor([S], device="cuda"), items, R,
                                        n_items=n_items)
    _, kept_ex, meta_ex = kernels.select_batch(raw_ex, "top_percent", k_top=K)
    kept_ex = kept_ex.cpu().numpy()
    gaps, refined = [], 0
    for b in range(B):
        ref_raw, ref_kept, dist = _oracle(q, k, v, b)
        np.testing.assert_allclose(raw[b], ref_raw, rtol=2e-5, atol=1e-12)
        np.testing.assert_allclose(raw_ex[b].cpu().numpy(), ref_raw, rtol=1e-12, atol=1e-18)
        m = np.sort(np.asarray(dist.masses))[::-1]
        gaps.append((m[K - 1] - m[K]) / m[K - 1])
        assert tuple(sorted(int(x) for x in kept_ex[b, :K])) == ref_kept
        if margin[b] > 1e-3:
            assert kept[b] == ref_kept, (b, margin[b])
        else:
            refined += 1
    print(f"unplanted: min K-boundary relative gap {min(gaps):.3e}, {refined}/{B} below the refinement margin")


def test_exact_ties_go_to_the_lower_index():
    """Round 25 strongest; rounds 3, 11, 17, 28 identical (copies of round 3) and
    second: K = 4 keeps {3, 11, 17, 25} and drops the tied 28 (stable order)."""
    def plant(b, kb, u):
        beta = 0.35 * np.sqrt(D)
        kb[25 * T:26 * T] += 1.4 * beta * u[None]
        kb[3 * T:4 * T] += beta * u[None]
        for r in (11, 17, 28):
            kb[r * T:(r + 1) * T] = kb[3 * T:4 * T]
    B = 3
    q, k, v = _dialogues(B, seed=77, plant=plant)
    raw, kept, _ = _gpu_scores(q, k, v)
    for b in range(B):
        assert raw[b, 3] == raw[b, 11] == raw[b, 17] == raw[b, 28], raw[b, [3, 11, 17, 28]]   # bit-identical
        ref_raw, ref_kept, _ = _oracle(q, k, v, b)
        assert ref_kept == (3, 11, 17, 25)
        assert kept[b] == ref_kept
        np.testing.assert_allclose(raw[b], ref_raw, rtol=2e-5, atol=1e-12)


def test_zero_mass_is_degenerate():
    """Every round inactive (all dropped): raw = 0, the distribution is
    degenerate (uniform) and the selector's fallback equals the reference's."""
    B = 2
    q, k, v = _dialogues(B, seed=5)
    active = np.zeros(R, bool)
    raw, kept, meta = _gpu_scores(q, k, v, active=active)
    assert not raw.any()
    for b in range(B):
        _, ref_kept, dist = _oracle(q, k, v, b, active=active)
        assert dist.degenerate and meta[1, b] == 1
        assert kept[b] == ref_kept


def test_exact_ties_multirow_prefill_scoring():
    """The same tie rule for a multi-row question (C3-style 512-row question,
    4 kv-heads x 7).  The tcgen05 prefill's fused Eq. 1 masses are fp32-class
    (identical rounds agree to ~1e-7, not bit for bit), so a tie at the K
    boundary shows up as a selection margin below the engines' refine threshold
    (EngineConfig.refine_margin, 1e-5), and the fp64 exact re-score (rk_round_scores_exact, what the engine
    then runs) gives bit-identical masses and keeps the lower indices."""
    from paper_2502_15294_b200.stats import build_round_items
    hq, hkv, d, nq, n_r, Tr = 28, 4, 128, 512, 16, 512
    hist = n_r * Tr
    s = hist + nq
    rng = np.random.default_rng(9)
    q = rng.standard_normal((nq, hq, d)).astype(np.float32)
    k = rng.standard_normal((s, hkv, d)).astype(np.float32)
    v = oatt.round_to_bf16(rng.standard_normal((s, hkv, d)).astype(np.float32))
    u = q.reshape(nq, hkv, hq // hkv, d).mean(axis=(0, 2))
    u /= np.linalg.norm(u, axis=-1, keepdims=True)
    beta = 0.3 * np.sqrt(d)
    k[9 * Tr:10 * Tr] += 1.4 * beta * u[None]
    k[2 * Tr:3 * Tr] += beta * u[None]
    for r in (5, 13):                        # 2, 5, 13 identical; K = 2 keeps {2, 9}
        k[r * Tr:(r + 1) * Tr] = k[2 * Tr:3 * Tr]
    k = oatt.round_to_bf16(k)
    qp, kp = np.arange(hist, s), np.arange(s)
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()  # noqa: E731
    bounds = [(r * Tr, (r + 1) * Tr, r) for r in range(n_r)] + [(hist, s, n_r)]
    items = torch.from_numpy(build_round_items(bounds, 1024)).cuda()
    _, raw, _ = kernels.prefill_attention(t(q), t(k).bfloat16(), t(v).bfloat16(), t(qp.astype(np.int64)),
                                          t(kp.astype(np.int64)), items=items, n_bins=n_r)
    margin = kernels.selection_margin(kernels.select_batch(raw[None], "top_percent", k_top=2)[0], "top_percent",
                                      k_top=2)
    raw = raw.cpu().numpy()
    np.testing.assert_allclose(raw[[5, 13]], raw[2], rtol=1e-6)
    from paper_2502_15294_b200.decode_engine import EngineConfig
    assert float(margin[0]) < EngineConfig.refine_margin, float(margin[0])   # -> the engine re-scores exactly
    exact = kernels.round_scores_exact(t(q)[None], t(k).bfloat16()[None], t(qp.astype(np.int64)), items[None],
                                       n_r).cpu().numpy()[0]
    assert exact[2] == exact[5] == exact[13], exact[[2, 5, 13]]
    # the fused masses are fp32-class: far inside the refine margin (measured <= 3e-8 on C3)
    np.testing.assert_allclose(raw, exact, rtol=1e-6)
    pol = orr.SelectionPolicy("top_percent", fraction=0.10)
    kept = orr.select(orr.normalize(exact), pol)
    _, cap = oatt.attention_forward_gqa(q, k, k, qp, kp, capture=True)
    rounds = [orr.Round(r, (r * Tr, r * Tr + 1), (r * Tr + 1, (r + 1) * Tr)) for r in range(n_r)]
    rounds.append(orr.Round(n_r, (hist, s), (s, s)))
    ref_raw = orr.aggregate_round_attention(cap, rounds, "question", n_r, row_offset=hist)
    ref_kept = orr.select(orr.normalize(ref_raw), pol)
    assert ref_kept == (2, 9) and kept == ref_kept
    np.testing.assert_allclose(raw, ref_raw, rtol=2e-5, atol=1e-9)
    # the scores-only form (rk_round_scores, the multi-row watershed scorer)
    from paper_2502_15294_b200 import stats
    raw2 = stats.round_scores(t(q), t(k).bfloat16(), qp, kp, bounds, n_r, chunk=1024, exact=False).cpu().numpy()
    assert raw2[2] == raw2[5] == raw2[13], raw2[[2, 5, 13]]
    assert orr.select(orr.normalize(raw2), pol) == ref_kept
    np.testing.assert_allclose(raw2, ref_raw, rtol=2e-5, atol=1e-9)
