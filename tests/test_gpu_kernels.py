"""GPU parity: librk kernels (through the C-ABI) against the oracle and the
reference's golden vectors.  Mirrors the reference conformance suite
(tests/test_backend.py:24-114) for the new backend."""

from __future__ import annotations

import numpy as np
import pytest

from conftest import load_kernel_cases, load_select_cases, load_stats_cases
from oracle import attention as oatt
from oracle import rounds as orr

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover - CPU container
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2502_15294_b200 import backend, kernels, selection, stats  # noqa: E402
from paper_2502_15294_b200.errors import DomainError, InvariantError  # noqa: E402

KERNEL = load_kernel_cases()


def _case(rng, n=5, s=12, heads=4, d_k=8, masked=False):
    q = rng.standard_normal((n, heads, d_k)).astype(np.float32)
    k = rng.standard_normal((s, heads, d_k)).astype(np.float32)
    v = rng.standard_normal((s, heads, d_k)).astype(np.float32)
    allowed = None
    if masked:
        allowed = rng.random(s) < 0.6
        allowed[s - n:] = True
    return q, k, v, np.arange(s - n, s), np.arange(s), allowed


# ----------------------------------------------------------------- kernel contract
@pytest.mark.parametrize("idx", range(len(KERNEL)))
def test_golden_attention_forward(idx):
    c = KERNEL[idx]
    out, scores = backend.attention_forward(c["q"], c["k"], c["v"], c["q_pos"], c["k_pos"],
                                            allowed=c["allowed"], capture=c["capture"])
    assert out.dtype == np.float32 and out.shape == c["out"].shape
    np.testing.assert_allclose(out, c["out"], rtol=1e-5, atol=1e-5)
    if c["capture"]:
        assert scores.dtype == np.float64
        np.testing.assert_allclose(scores, c["scores"], rtol=1e-5, atol=1e-7)
        np.testing.assert_array_equal(scores == 0.0, c["scores"] == 0.0)   # exact causal zeros
    else:
        assert scores is None


def test_single_query_single_key(rng):
    q, k, v = (rng.standard_normal((1, 1, 2)).astype(np.float32) for _ in range(3))
    out, scores = backend.attention_forward(q, k, v, np.array([0]), np.array([0]), capture=True)
    np.testing.assert_array_equal(scores, [[1.0]])
    np.testing.assert_allclose(out[0], v.reshape(-1), rtol=1e-6)


def test_rows_normalized_and_causal(rng):
    q, k, v, qp, kp, _ = _case(rng)
    _, scores = backend.attention_forward(q, k, v, qp, kp, capture=True)
    np.testing.assert_allclose(scores.sum(axis=1), 1.0, atol=1e-12)
    for i, p in enumerate(qp):
        assert np.all(scores[i, p + 1:] == 0.0)


def test_contract_edges(rng):
    q, k, v, qp, kp, _ = _case(rng)
    out, scores = backend.attention_forward(q[:0], k, v, np.zeros(0, np.int64), kp, capture=True)
    assert out.shape == (0, 32) and scores.shape == (0, 12)
    assert backend.attention_forward(q, k, v, qp, kp)[1] is None
    with pytest.raises(InvariantError, match="no visible key"):
        backend.attention_forward(q, k, v, qp, kp, allowed=np.zeros(12, dtype=bool))
    with pytest.raises(DomainError):
        backend.attention_forward(q, k, v[:, :2], qp, kp)
    with pytest.raises(DomainError):
        backend.attention_forward(q, k, v, qp[:2], kp)
    assert backend.BACKEND_NAME == "cuda"
    assert backend.available_backends() == {"cuda": backend}


@pytest.mark.parametrize("G,d,dtype", [(4, 128, "bf16"), (7, 128, "bf16"), (4, 64, "f32"), (2, 40, "f32"),
                                       (8, 128, "f32"), (1, 256, "bf16")])
def test_gqa_masked_vs_oracle(rng, G, d, dtype):
    hkv, n, s = 2, 6, 700
    q = rng.standard_normal((n, hkv * G, d)).astype(np.float32)
    k = rng.standard_normal((s, hkv, d)).astype(np.float32)
    v = rng.standard_normal((s, hkv, d)).astype(np.float32)
    if dtype == "bf16":
        k, v = oatt.round_to_bf16(k), oatt.round_to_bf16(v)
    allowed = rng.random(s) < 0.7
    allowed[s - n:] = True
    qp, kp = np.arange(s - n, s), np.arange(s)
    ref_out, ref_sc = oatt.attention_forward_gqa(q, k, v, qp, kp, allowed=allowed, capture=True)
    tk = torch.from_numpy(k).cuda()
    tv = torch.from_numpy(v).cuda()
    if dtype == "bf16":
        tk, tv = tk.bfloat16(), tv.bfloat16()
    out, sc = backend.attention_forward_gqa(torch.from_numpy(q).cuda(), tk, tv, torch.from_numpy(qp),
                                            torch.from_numpy(kp), allowed=torch.from_numpy(allowed), capture=True)
    np.testing.assert_allclose(out.cpu().numpy(), ref_out, rtol=1e-4, atol=2e-5)
    np.testing.assert_allclose(sc.cpu().numpy(), ref_sc, rtol=1e-4, atol=1e-8)


# ----------------------------------------------------------------- decode
@pytest.mark.parametrize("G,d,dtype", [(4, 128, torch.bfloat16), (7, 128, torch.bfloat16),
                                       (4, 128, torch.float32), (1, 64, torch.float32), (8, 64, torch.bfloat16),
                                       (2, 48, torch.float32)])
def test_decode_append_vs_oracle(rng, G, d, dtype):
    B, hkv, cap = 3, 4 if G < 7 else 2, 3000
    lens = np.array([2999, 17, 1024])
    kc = torch.randn(B, cap + 1, hkv, d, device="cuda").to(dtype)
    vc = torch.randn(B, cap + 1, hkv, d, device="cuda").to(dtype)
    q = torch.randn(B, hkv * G, d, device="cuda")
    kn = torch.randn(B, hkv, d, device="cuda").to(dtype)
    vn = torch.randn(B, hkv, d, device="cuda").to(dtype)
    sl = torch.from_numpy(lens.astype(np.int32)).cuda()
    out = kernels.decode_attention(q, kc, vc, sl, int(lens.max()) + 1, k_new=kn, v_new=vn)
    for b in range(B):
        L = lens[b]
        kk = kc[b, : L + 1].float().cpu().numpy()
        vv = vc[b, : L + 1].float().cpu().numpy()
        np.testing.assert_array_equal(kk[L], kn[b].float().cpu().numpy())     # appended
        np.testing.assert_array_equal(vv[L], vn[b].float().cpu().numpy())
        ref, _ = oatt.attention_forward_gqa(q[b:b + 1].cpu().numpy(), kk, vv, [L], np.arange(L + 1))
        got = out[b].reshape(1, -1).cpu().numpy()
        err = np.abs(got - ref).max() / np.abs(ref).max()
        assert err < 1e-5, err          # spec: 1e-3 relative
    assert torch.equal(sl.cpu(), torch.from_numpy(lens.astype(np.int32)))


@pytest.mark.parametrize("lens", [
    [2999, 17, 1024, 1, 700, 2048, 5, 333, 1500, 64, 2999, 900],     # ragged, a dialogue spans 1..many CTAs
    [3, 1, 2, 5, 4, 1, 2, 3, 1],                                       # fewer keys than CTAs (sparse ranges)
    [2999] * 16,                                                       # the bench's 16-dialogue group shape
])
def test_decode_larger_batches_vs_oracle(rng, lens):
    """B >= 8 ragged / sparse / bench-shaped batches: persistent split over the
    concatenated key ranges + merge; repeated calls and a different shape on
    the same workspace arena give identical results."""
    B, hkv, G, d, cap = len(lens), 8, 4, 128, 3000
    lens = np.array(lens)
    torch.manual_seed(len(lens))
    kc = torch.randn(B, cap + 1, hkv, d, device="cuda").bfloat16()
    vc = torch.randn(B, cap + 1, hkv, d, device="cuda").bfloat16()
    q = torch.randn(B, hkv * G, d, device="cuda")
    kn = torch.randn(B, hkv, d, device="cuda").bfloat16()
    vn = torch.randn(B, hkv, d, device="cuda").bfloat16()
    sl = torch.from_numpy(lens.astype(np.int32)).cuda()
    ws = kernels.decode_workspace(B, hkv * G, hkv, d, 592, "cuda", tag="batch_test")
    outs = []
    for rep in range(3):
        outs.append(kernels.decode_attention(q, kc, vc, sl, int(lens.max()) + 1, k_new=kn, v_new=vn, ws=ws).clone())
        # a different (smaller) batch on the same arena between calls
        kernels.decode_attention(q[:9], kc[:9], vc[:9], sl[:9], int(lens[:9].max()) + 1, k_new=kn[:9],
                                 v_new=vn[:9], ws=ws)
    torch.cuda.synchronize()
    for rep in range(1, 3):
        assert torch.equal(outs[rep], outs[0])
    out = outs[0]
    for b in range(B):
        L = lens[b]
        kk = kc[b, : L + 1].float().cpu().numpy()
        vv = vc[b, : L + 1].float().cpu().numpy()
        ref, _ = oatt.attention_forward_gqa(q[b:b + 1].cpu().numpy(), kk, vv, [L], np.arange(L + 1))
        err = np.abs(out[b].reshape(1, -1).cpu().numpy() - ref).max() / np.abs(ref).max()
        # q and P carry ~16 mantissa bits (bf16 hi + lo): ~5e-6 typical over 12 seeds, 8e-6 worst
        assert err < 2e-5, (b, err)


def test_decode_advance_lengths():
    sl = torch.tensor([3, 5], dtype=torch.int32, device="cuda")
    kernels.advance_lengths(sl, 2)
    assert sl.tolist() == [5, 7]


# ----------------------------------------------------------------- scoring
def _rounds_layout(rng, n_rounds, lo=50, hi=400):
    lens = rng.integers(lo, hi, size=n_rounds)
    starts = np.concatenate([[0], np.cumsum(lens)])
    return lens, starts


@pytest.mark.parametrize("n_q,G,dtype", [(1, 4, torch.bfloat16), (7, 4, torch.float32), (33, 1, torch.float32),
                                         (5, 7, torch.bfloat16),
                                         # >= 64 stacked rows, bf16, d=128: the tcgen05 scorer (scores-only prefill_tc.cu)
                                         (64, 4, torch.bfloat16), (100, 7, torch.bfloat16), (130, 1, torch.bfloat16)])
def test_round_scores_vs_capture_aggregate(rng, n_q, G, dtype):
    n_rounds, hkv, d = 9, 2, 128
    lens, starts = _rounds_layout(rng, n_rounds)
    hist = int(starts[-1])
    s = hist + n_q
    q = rng.standard_normal((n_q, hkv * G, d)).astype(np.float32)
    k = rng.standard_normal((s, hkv, d)).astype(np.float32)
    if dtype == torch.bfloat16:
        k = oatt.round_to_bf16(k)
    qp = np.arange(hist, s)
    kp = np.arange(s)
    _, cap = oatt.attention_forward_gqa(q, k, k, qp, kp, capture=True)
    rounds = [orr.Round(m, (int(starts[m]), int(starts[m]) + 3), (int(starts[m]) + 3, int(starts[m + 1])))
              for m in range(n_rounds)]
    rounds.append(orr.Round(n_rounds, (hist, s), (s, s)))
    active = [m for m in range(n_rounds) if m != 4]
    ref = orr.aggregate_round_attention(cap, rounds, "question", n_rounds, active_rounds=active, row_offset=hist)
    bounds = [(int(starts[m]), int(starts[m + 1]), m) for m in range(n_rounds)] + [(hist, s, n_rounds)]
    mask = [m in active for m in range(n_rounds)]
    raw = stats.round_scores(torch.from_numpy(q).cuda(), torch.from_numpy(k).cuda().to(dtype), qp, kp, bounds,
                             n_rounds, active=mask, chunk=128)
    np.testing.assert_allclose(raw.cpu().numpy(), ref, rtol=2e-5, atol=1e-9)


@pytest.mark.parametrize("hkv,G", [(8, 4), (4, 7), (2, 4)])
def test_fused_decode_scoring_vs_oracle(rng, hkv, G):
    """Layer Lw-1 decode with round-aligned items = attention output + Eq. 1."""
    B, d = 2, 128
    n_rounds = 12
    per_b = []
    lens_all = []
    for b in range(B):
        lens, starts = _rounds_layout(rng, n_rounds, 100, 700)
        per_b.append(starts)
        lens_all.append(int(starts[-1]))
    cap = max(lens_all) + 1
    kc = torch.randn(B, cap, hkv, d, device="cuda").bfloat16()
    vc = torch.randn(B, cap, hkv, d, device="cuda").bfloat16()
    q = torch.randn(B, hkv * G, d, device="cuda")
    kn = torch.randn(B, hkv, d, device="cuda").bfloat16()
    vn = torch.randn(B, hkv, d, device="cuda").bfloat16()
    sl = torch.tensor(lens_all, dtype=torch.int32, device="cuda")
    bounds = [[(int(st[m]), int(st[m + 1]), m) for m in range(n_rounds)] + [(int(st[-1]), int(st[-1]) + 1, n_rounds)]
              for st in per_b]
    items, n_items = kernels.items_tensor(bounds, 256, "cuda")
    ws = kernels.decode_workspace(B, hkv * G, hkv, d, items.shape[1], "cuda", tag="t_fused")
    out = kernels.decode_attention(q, kc, vc, sl, cap, k_new=kn, v_new=vn, items=items, n_items=n_items, ws=ws)
    raw = kernels.decode_scores_finalize(B, hkv * G, hkv, d, items, n_items, n_rounds, ws, kv_dtype=torch.bfloat16)
    for b in range(B):
        L = lens_all[b]
        kk = kc[b, : L + 1].float().cpu().numpy()
        vv = vc[b, : L + 1].float().cpu().numpy()
        ref_out, capm = oatt.attention_forward_gqa(q[b:b + 1].cpu().numpy(), kk, vv, [L], np.arange(L + 1),
                                                   capture=True)
        np.testing.assert_allclose(out[b].reshape(1, -1).cpu().numpy(), ref_out, rtol=1e-4, atol=1e-5)
        st = per_b[b]
        ref_raw = np.array([capm[0, st[m]:st[m + 1]].sum() for m in range(n_rounds)])
        np.testing.assert_allclose(raw[b].cpu().numpy(), ref_raw, rtol=2e-5, atol=1e-10)


# ----------------------------------------------------------------- stats + selection (bit-exact)
def test_golden_aggregate_and_normalize():
    for case in load_stats_cases():
        rounds = orr.make_rounds([tuple(x) for x in case["layout"]])
        n = len(rounds) - 1
        raw = stats.aggregate_round_attention(case["scores"], rounds, "question", n,
                                              active_rounds=list(case["active"]),
                                              row_offset=int(case["row_offset"]))
        np.testing.assert_allclose(raw, case["raw"], rtol=1e-13, atol=1e-15)
        dist = stats.normalize(case["raw"], round_indices=list(case["active"]))
        np.testing.assert_array_equal(dist.masses, case["masses"])        # bit-exact
        assert dist.degenerate == bool(case["degenerate"])


def test_golden_selection_bit_exact():
    cases = load_select_cases()
    for c in cases:
        dist = stats.normalize(c["raw"])
        np.testing.assert_array_equal(dist.masses, c["masses"])
        assert dist.degenerate == c["degenerate"]
        for r in c["results"]:
            pol = selection.SelectionPolicy(kind=r["kind"], **r["params"])
            res = selection.select(dist, pol)
            assert list(res.kept) == r["kept"], (r, c["raw"][:6])


def test_selection_errors_and_empty():
    with pytest.raises(DomainError, match="non-negative"):
        stats.normalize(np.array([0.5, -0.1]))
    d0 = stats.normalize(np.zeros(0))
    assert selection.select(d0, selection.SelectionPolicy()).kept == ()
    with pytest.raises(DomainError):
        selection.SelectionPolicy(kind="token_baseline").__class__  # valid kind
        selection.select(stats.normalize(np.ones(3)), selection.SelectionPolicy(kind="token_baseline"))


@pytest.mark.parametrize("idx", [0, 3, 7, 25, 27])
def test_engine_attention_layer_on_golden(idx):
    """engine.attention_layer (engine.py:120-143): flat (rows, d_model) operands,
    default causal positions, capture on by default — equals the reference's
    attention_forward golden output / scores for the same case."""
    from paper_2502_15294_b200.engine import attention_layer
    c = KERNEL[idx]
    n, h, d = c["q"].shape
    s = c["k"].shape[0]
    flat = lambda x: x.reshape(x.shape[0], h * d)  # noqa: E731
    out, scores = attention_layer(flat(c["q"]), flat(c["k"]), flat(c["v"]), num_heads=h, allowed=c["allowed"])
    assert np.array_equal(c["q_pos"], np.arange(s - n, s)) and np.array_equal(c["k_pos"], np.arange(s))
    np.testing.assert_allclose(out, c["out"], rtol=1e-5, atol=1e-5)
    if c["capture"]:
        np.testing.assert_allclose(scores, c["scores"], rtol=1e-5, atol=1e-7)
    with pytest.raises(DomainError):
        attention_layer(c["q"], flat(c["k"]), flat(c["v"]), num_heads=h)


def test_backend_contract_edge_cases_like_reference(rng):
    """The reference's backend contract tests (test_backend.py:26-90) against
    this backend: one query / one key, rows normalised and causal, empty query
    set, capture off -> None, no visible key -> InvariantError("...no visible
    key..."), shape mismatches -> DomainError."""
    q, k, v, q_pos, k_pos, _ = _case(rng, n=5, s=12, heads=4, d_k=8)
    o1, s1 = backend.attention_forward(q[:1], k[:1], v[:1], np.array([0]), np.array([0]), capture=True)
    np.testing.assert_allclose(o1.reshape(1, 4, 8), v[:1], rtol=1e-6, atol=1e-6)   # one key: out = v
    assert s1.shape == (1, 1) and s1[0, 0] == 1.0
    out, sc = backend.attention_forward(q, k, v, q_pos, k_pos, capture=True)
    np.testing.assert_allclose(sc.sum(axis=1), 1.0, rtol=1e-12, atol=1e-12)
    for i, p in enumerate(q_pos):
        assert np.all(sc[i, k_pos > p] == 0.0)
    oe, se = backend.attention_forward(q[:0], k, v, np.zeros(0, dtype=np.int64), k_pos, capture=True)
    assert oe.shape == (0, 32) and se.shape == (0, 12)
    assert backend.attention_forward(q, k, v, q_pos, k_pos)[1] is None
    with pytest.raises(InvariantError, match="no visible key"):
        backend.attention_forward(q, k, v, q_pos, k_pos, allowed=np.zeros(12, dtype=bool))
    with pytest.raises(DomainError):
        backend.attention_forward(q, k, v[:, :2], q_pos, k_pos)
    with pytest.raises(DomainError):
        backend.attention_forward(q, k, v, q_pos[:2], k_pos)


def test_normalize_properties_like_reference(rng):
    """stats.normalize (device) on the reference's test_stats.TestNormalize cases."""
    d = stats.normalize(np.array([2.0, 2.0]))
    np.testing.assert_allclose(d.masses, [0.5, 0.5])
    assert not d.degenerate
    d = stats.normalize(np.zeros(3))
    np.testing.assert_allclose(d.masses, [1 / 3] * 3)
    assert d.degenerate
    np.testing.assert_allclose(stats.normalize(np.array([0.75, 0.25])).masses, [0.75, 0.25])
    with pytest.raises(DomainError, match="non-negative"):
        stats.normalize(np.array([0.5, -0.1]))
    for _ in range(50):
        raw = rng.random(int(rng.integers(1, 30))) * rng.integers(1, 100)
        assert abs(np.asarray(stats.normalize(raw).masses).sum() - 1.0) <= 1e-6


def test_aggregate_round_attention_like_reference(rng):
    """stats.aggregate_round_attention (rk_aggregate_rounds) on the reference's
    test_stats.TestAggregate cases: hand-built rows, split across rounds, zero
    block, 50 random matrices vs the double-loop oracle (both segments),
    row_offset mapping, missing rows / empty span rejected."""
    agg = stats.aggregate_round_attention

    def causal(s):
        m = np.zeros((s, s))
        for i in range(s):
            r = rng.random(i + 1)
            m[i, :i + 1] = r / r.sum()
        return m

    def brute(m, rounds, seg, n, k):
        rnd = rounds[n]
        span = rnd.q_span if seg == "question" else rnd.a_span
        cols = list(range(*rounds[k].q_span)) + list(range(*rounds[k].a_span))
        return sum(float(m[i][j]) for i in range(*span) for j in cols)

    rounds = orr.make_rounds([(2, 1), (1, 0)])
    mat = np.zeros((4, 4))
    mat[3, :4] = 0.25
    for i in range(3):
        mat[i, :i + 1] = 1.0 / (i + 1)
    np.testing.assert_allclose(agg(mat, rounds, "question", 1), [0.75])
    rounds = orr.make_rounds([(2, 1), (1, 0), (1, 0)])
    mat = np.zeros((5, 5))
    mat[4, :4] = 0.25
    for i in range(4):
        mat[i, :i + 1] = 1.0 / (i + 1)
    np.testing.assert_allclose(agg(mat, rounds, "question", 2), [0.75, 0.25])
    rounds = orr.make_rounds([(1, 1), (1, 1)])
    mat = np.zeros((4, 4))
    mat[2, 2] = mat[3, 3] = 1.0
    np.testing.assert_array_equal(agg(mat, rounds, "question", 1), [0.0])
    for _ in range(50):
        layout = [(int(rng.integers(1, 4)), int(rng.integers(1, 4))) for _ in range(int(rng.integers(2, 5)))]
        rounds = orr.make_rounds(layout)
        n = len(rounds) - 1
        mat = causal(rounds[-1].end)
        for seg in ("question", "answer"):
            raw = agg(mat, rounds, seg, n)
            for k in range(n):
                assert abs(raw[k] - brute(mat, rounds, seg, n, k)) <= 1e-9
    rounds = orr.make_rounds([(2, 2), (3, 0)])
    full = causal(7)
    np.testing.assert_allclose(agg(full, rounds, "question", 1), agg(full[4:7], rounds, "question", 1, row_offset=4),
                               atol=1e-12)
    with pytest.raises(DomainError, match="absent"):
        agg(full[5:], rounds, "question", 1, row_offset=5)
    with pytest.raises(DomainError, match="empty"):
        agg(np.zeros((7, 7)), rounds, "answer", 1)
