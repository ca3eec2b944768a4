"""Bit-exact kept rounds by construction (SURVEY.md §7 hard part 1, VERDICT r1
"next" item 1): the exact watershed scorer (rk_round_scores_exact — the
reference kernel's fp64 arithmetic, _attn_ext.pyx:52-76,113-114 + stats.py:59-94)
followed by the device selector must reproduce the reference's kept set with
NO tolerance escape:

  * golden kernel cases (captures produced by the reference itself);
  * unplanted keys at C2 shapes (hard parity, small K-boundary gaps);
  * exact ties (duplicated rounds straddling K -> lower index);
  * full-size C3 (64 rounds x 1 K keys, 512-row question, Hq 28 / Hkv 4, K = 7);
  * full-size C4 (128 rounds x 1 K keys, 1-row question, 16 dialogues, K = 13);

raw masses within 1e-12 relative of the oracle (oracle/attn_ref.c's
`attn_ref_round_masses`: the reference's capture arithmetic), kept sets equal,
and the K-boundary margin of every case recorded in profiles/ by the bench.
The fp32-class fused scorers are checked for the margin contract: their kept
set equals the reference's whenever the margin exceeds the refinement
threshold, and the engines re-score exactly below it."""

from __future__ import annotations

import concurrent.futures as cf
import os

import numpy as np
import pytest

from conftest import load_kernel_cases
from oracle import cref
from oracle import rounds as orr

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2502_15294_b200 import kernels  # noqa: E402
from paper_2502_15294_b200.stats import build_round_items  # noqa: E402

POLICY = orr.SelectionPolicy("top_percent", fraction=0.10)
THREADS = os.cpu_count() or 1


def _rel_gap(masses, K):
    m = np.sort(np.asarray(masses))[::-1]
    if K >= len(m):
        return np.inf
    return (m[K - 1] - m[K]) / m[K - 1] if m[K - 1] > 0 else 0.0


def _bf16(t):
    return t.to(torch.bfloat16)


def _select(raw_dev, K):
    masses, kept, meta = kernels.select_batch(raw_dev, "top_percent", k_top=K)
    margin = kernels.selection_margin(masses, "top_percent", k_top=K)
    torch.cuda.synchronize()
    n = meta[0].cpu().numpy()
    return ([tuple(sorted(int(x) for x in kept[b, :n[b]].cpu().numpy())) for b in range(raw_dev.shape[0])],
            margin.cpu().numpy())


def test_exact_scorer_matches_reference_captures():
    """Golden kernel cases with capture=True and no mask (the reference's own
    capture matrices): keys split into bins, bin masses from the reference's
    capture vs the exact scorer, 1e-12 relative."""
    n_done = 0
    for c in load_kernel_cases():
        if not c["capture"] or c["allowed"] is not None or c["q"].shape[0] == 0:
            continue
        q, k = c["q"], c["k"]
        n, hq, d = q.shape
        s = k.shape[0]
        if d % 8 or s < 4:
            continue
        kp = c["k_pos"].astype(np.int64)
        if not np.all(np.diff(kp) > 0):
            continue
        cuts = np.linspace(0, s, 5).astype(int)
        bounds = [(int(cuts[i]), int(cuts[i + 1]), i) for i in range(4)]
        n_bins = 3                                    # the last bin stands for the current question
        ref = np.array([c["scores"][:, lo:hi].sum() for lo, hi, _ in bounds[:n_bins]])
        items = torch.from_numpy(build_round_items(bounds, 64)).cuda()[None]
        tq = torch.from_numpy(np.ascontiguousarray(q)).cuda()[None]
        tk = torch.from_numpy(np.ascontiguousarray(k)).cuda()[None]
        if c["bf16"]:
            tk = _bf16(tk)
        raw = kernels.round_scores_exact(tq, tk, torch.from_numpy(c["q_pos"].astype(np.int64)).cuda(), items,
                                         n_bins, k_pos=torch.from_numpy(kp).cuda()).cpu().numpy()[0]
        np.testing.assert_allclose(raw, ref, rtol=1e-12, atol=1e-15)
        n_done += 1
    assert n_done >= 5


R2, T2, HKV2, G2, D2 = 32, 512, 8, 4, 128


def _c2_batch(B, seed, plant=None):
    g = torch.Generator(device="cuda").manual_seed(seed)
    S = R2 * T2 + 1
    q = torch.randn((B, 1, HKV2 * G2, D2), generator=g, device="cuda")
    k = torch.randn((B, S, HKV2, D2), generator=g, device="cuda")
    if plant:
        plant(q, k)
    return q, _bf16(k)


def _c2_items(B):
    S = R2 * T2
    bounds = [[(m * T2, (m + 1) * T2, m) for m in range(R2)] + [(S, S + 1, R2)]] * B
    return kernels.items_tensor(bounds, 1024, "cuda")


def _oracle_many(jobs):
    """[(q (n,Hq,d), k (S,Hkv,d), q_pos, k_pos, spans, n_bins)] -> raw per job (threads over jobs)."""
    per = max(1, THREADS // max(1, len(jobs)))
    with cf.ThreadPoolExecutor(max_workers=min(THREADS, len(jobs))) as ex:
        return list(ex.map(lambda j: cref.round_masses(*j, threads=per), jobs))


def _c2_check(q, k, K, fraction=0.10):
    B = q.shape[0]
    S = R2 * T2 + 1
    items, n_items = _c2_items(B)
    raw = kernels.round_scores_exact(q, k, torch.tensor([S - 1], device="cuda"), items, R2, n_items=n_items)
    kept, margin = _select(raw, K)
    raw = raw.cpu().numpy()
    spans = [(m * T2, (m + 1) * T2, m) for m in range(R2)]
    jobs = [(q[b].cpu().numpy(), k[b].float().cpu().numpy(), [S - 1], np.arange(S), spans, R2) for b in range(B)]
    refs = _oracle_many(jobs)
    gaps = []
    for b in range(B):
        np.testing.assert_allclose(raw[b], refs[b], rtol=1e-12, atol=1e-18)
        want = orr.select(orr.normalize(refs[b]), orr.SelectionPolicy("top_percent", fraction=fraction))
        assert kept[b] == want, (b, kept[b], want, _rel_gap(orr.normalize(refs[b]).masses, K))
        gaps.append(_rel_gap(orr.normalize(refs[b]).masses, K))
        assert abs(margin[b] - gaps[-1]) <= 1e-9 * max(1.0, gaps[-1])
    return min(gaps)


def test_unplanted_c2_zero_tolerance():
    """No planted relevance: K-boundary gaps are small; kept sets must be equal
    in every dialogue (no tolerance escape)."""
    K = orr.top_k_count(R2, 0.10, 1)
    q, k = _c2_batch(16, seed=2002)
    g = _c2_check(q, k, K)
    print(f"unplanted C2: min K-boundary relative gap {g:.3e}")


def test_near_tie_c2_zero_tolerance():
    """Rounds 7 and 19 hold the same keys except one row (a near tie at the K
    boundary, gap ~1e-6..1e-9): the fp64 scorer still picks the reference's."""
    def plant(q, k):
        u = q[:, 0].view(-1, HKV2, G2, D2).mean(dim=2)
        u = u / u.norm(dim=-1, keepdim=True)
        k[:, 3 * T2:4 * T2] += 0.5 * (D2 ** 0.5) * u[:, None]
        k[:, 7 * T2:8 * T2] += 0.3 * (D2 ** 0.5) * u[:, None]
        k[:, 19 * T2:20 * T2] = k[:, 7 * T2:8 * T2]
        k[:, 19 * T2 + 5] += 1e-3 * torch.randn_like(k[:, 19 * T2 + 5])
    K = orr.top_k_count(R2, 0.05, 1)       # 2: round 3 and one of the near-tied 7 / 19
    q, k = _c2_batch(6, seed=31, plant=plant)
    g = _c2_check(q, k, K, fraction=0.05)
    print(f"near-tie C2: min gap {g:.3e}")


def test_exact_ties_c2_lower_index():
    """Rounds 3, 11, 17, 28 identical and second strongest after 25: K = 4 keeps
    {3, 11, 17, 25}; the duplicated rounds' masses are bit-identical."""
    def plant(q, k):
        u = q[:, 0].view(-1, HKV2, G2, D2).mean(dim=2)
        u = u / u.norm(dim=-1, keepdim=True)
        beta = 0.35 * D2 ** 0.5
        k[:, 25 * T2:26 * T2] += 1.4 * beta * u[:, None]
        k[:, 3 * T2:4 * T2] += beta * u[:, None]
        for r in (11, 17, 28):
            k[:, r * T2:(r + 1) * T2] = k[:, 3 * T2:4 * T2]
    K = orr.top_k_count(R2, 0.10, 1)
    q, k = _c2_batch(3, seed=77, plant=plant)
    items, n_items = _c2_items(3)
    S = R2 * T2 + 1
    raw = kernels.round_scores_exact(q, k, torch.tensor([S - 1], device="cuda"), items, R2, n_items=n_items)
    r = raw.cpu().numpy()
    for b in range(3):
        assert r[b, 3] == r[b, 11] == r[b, 17] == r[b, 28], r[b, [3, 11, 17, 28]]
    kept, margin = _select(raw, K)
    assert all(kk == (3, 11, 17, 25) for kk in kept), kept
    assert (margin == 0).all()          # the tie straddles K: decided by index
    _c2_check(q, k, K)


def test_c3_full_size_512_row_question():
    """C3 at full size: Qwen2-7B-shaped (Hq 28, Hkv 4, d 128), 64 rounds x 1024
    keys, a 512-row question, K = 7.  The exact scorer's raw masses (1e-12) and
    kept set equal the oracle's; the tcgen05 fused prefill scoring gives the
    same kept set whenever its margin clears the engines' 1e-3 threshold."""
    R, T, hq, hkv, d, nq = 64, 1024, 28, 4, 128, 512
    hist = R * T
    s = hist + nq
    K = orr.top_k_count(R, 0.10, 1)
    g = torch.Generator(device="cuda").manual_seed(3303)
    q = torch.randn((nq, hq, d), generator=g, device="cuda")
    k = torch.randn((s, hkv, d), generator=g, device="cuda")
    v = torch.randn((s, hkv, d), generator=g, device="cuda")
    u = q.view(nq, hkv, hq // hkv, d).mean(dim=(0, 2))
    u = u / u.norm(dim=-1, keepdim=True)
    for r, beta in ((5, 0.05), (40, 0.045), (22, 0.04)):       # mild relevance: gaps of a few 1e-2
        k[r * T:(r + 1) * T] += beta * d ** 0.5 * u[None]
    k, v = _bf16(k), _bf16(v)
    qp = torch.arange(hist, s, device="cuda")
    kp = torch.arange(s, device="cuda")
    bounds = [(r * T, (r + 1) * T, r) for r in range(R)] + [(hist, s, R)]
    items = torch.from_numpy(build_round_items(bounds, 1024)).cuda()
    raw_ex = kernels.round_scores_exact(q[None], k[None], qp, items[None], R)
    kept_ex, margin_ex = _select(raw_ex, K)
    _, raw_tc, _ = kernels.prefill_attention(q, k, v, qp, kp, items=items, n_bins=R)
    kept_tc, margin_tc = _select(raw_tc[None], K)
    ref = cref.round_masses(q.cpu().numpy(), k.float().cpu().numpy(), qp.cpu().numpy(), kp.cpu().numpy(),
                            bounds[:R], R, threads=THREADS)
    np.testing.assert_allclose(raw_ex.cpu().numpy()[0], ref, rtol=1e-12, atol=1e-15)
    want = orr.select(orr.normalize(ref), POLICY)
    assert kept_ex[0] == want
    gap = _rel_gap(orr.normalize(ref).masses, K)
    assert abs(margin_ex[0] - gap) <= 1e-9
    np.testing.assert_allclose(raw_tc.cpu().numpy(), ref, rtol=2e-5)
    if margin_tc[0] > 1e-3:
        assert kept_tc[0] == want
    print(f"C3 512-row: kept {want}, K-boundary gap {gap:.3e} (tcgen05 margin {margin_tc[0]:.3e})")


def test_c4_full_size_16_dialogues():
    """C4 at full size: Llama-3-8B-shaped, 128 rounds x 1024 keys (131 K), one
    decode-token question per dialogue, 16 dialogues, K = 13 — the exact
    scorer's kept sets equal the oracle's in every dialogue, raw 1e-12."""
    R, T, hkv, G, d, B = 128, 1024, 8, 4, 128, 16
    S = R * T + 1
    K = orr.top_k_count(R, 0.10, 1)
    g = torch.Generator(device="cuda").manual_seed(4404)
    q = torch.randn((B, 1, hkv * G, d), generator=g, device="cuda")
    k = _bf16(torch.randn((B, S, hkv, d), generator=g, device="cuda"))
    bounds = [[(m * T, (m + 1) * T, m) for m in range(R)] + [(S - 1, S, R)]] * B
    items, n_items = kernels.items_tensor(bounds, 1024, "cuda")
    raw = kernels.round_scores_exact(q, k, torch.tensor([S - 1], device="cuda"), items, R, n_items=n_items)
    kept, margin = _select(raw, K)
    raw = raw.cpu().numpy()
    spans = [(m * T, (m + 1) * T, m) for m in range(R)]
    refs = []
    for b0 in range(0, B, 4):               # bounded host memory: 4 dialogues' fp32 keys at a time
        jobs = [(q[b].cpu().numpy(), k[b].float().cpu().numpy(), [S - 1], np.arange(S), spans, R)
                for b in range(b0, b0 + 4)]
        refs += _oracle_many(jobs)
    gaps = []
    for b in range(B):
        np.testing.assert_allclose(raw[b], refs[b], rtol=1e-12, atol=1e-18)
        want = orr.select(orr.normalize(refs[b]), POLICY)
        assert kept[b] == want, b
        gaps.append(_rel_gap(orr.normalize(refs[b]).masses, K))
    print(f"C4: min K-boundary gap over 16 dialogues {min(gaps):.3e}")


@pytest.mark.parametrize("n_q,hq,hkv,d,R,T", [(1, 32, 8, 128, 32, 512), (4, 28, 4, 128, 16, 256),
                                              (7, 8, 8, 64, 8, 128), (1, 8, 2, 64, 12, 97)])
def test_exact_pre_scorer_matches_oracle(n_q, hq, hkv, d, R, T):
    """capture_mode="pre" (engine.py:187-200) on rk_round_scores_exact_pre: one
    softmax per row over the head-summed fp64 logits / (Hq sqrt(d)); Eq. 1 masses
    vs the oracle's capture_pre + aggregate within 1e-12, kept sets equal."""
    from oracle import attention as oatt
    rng = np.random.default_rng(n_q * 1000 + hq + R)
    B = 2
    hist = R * T
    s = hist + n_q
    k = oatt.round_to_bf16(rng.standard_normal((B, s, hkv, d)).astype(np.float32))
    q = rng.standard_normal((B, n_q, hq, d)).astype(np.float32)
    q_pos = np.arange(hist, hist + n_q, dtype=np.int64)
    bounds = [(r * T, (r + 1) * T, r) for r in range(R)] + [(hist, s, R)]
    items = build_round_items(bounds, 256)
    it = torch.from_numpy(np.stack([items] * B)).cuda()
    raw = kernels.round_scores_exact(torch.from_numpy(q).cuda(), _bf16(torch.from_numpy(k).cuda()),
                                     torch.from_numpy(q_pos).cuda(), it, R, capture_mode="pre")
    K = orr.top_k_count(R, 0.10, 1)
    kept, _ = _select(raw, K)
    raw = raw.cpu().numpy()
    for b in range(B):
        cap = oatt.capture_pre(q[b], k[b], q_pos, np.arange(s))
        want = np.array([cap[:, r * T:(r + 1) * T].sum() for r in range(R)])
        np.testing.assert_allclose(raw[b], want, rtol=1e-12, atol=0)
        dist = orr.normalize(want)
        assert kept[b] == orr.select(dist, POLICY), (b, kept[b])


def test_exact_pre_differs_from_post():
    """The two capture modes are different statistics (guards a silent mode mix-up)."""
    rng = np.random.default_rng(5)
    R, T, hq, hkv, d = 8, 64, 8, 2, 64
    s = R * T + 1
    k = _bf16(torch.from_numpy(rng.standard_normal((1, s, hkv, d)).astype(np.float32)).cuda())
    q = torch.from_numpy(rng.standard_normal((1, 1, hq, d)).astype(np.float32)).cuda()
    qp = torch.tensor([R * T], dtype=torch.int64, device="cuda")
    it = torch.from_numpy(build_round_items([(r * T, (r + 1) * T, r) for r in range(R)] + [(R * T, s, R)], 256)
                          )[None].cuda()
    post = kernels.round_scores_exact(q, k, qp, it, R).cpu().numpy()
    pre = kernels.round_scores_exact(q, k, qp, it, R, capture_mode="pre").cpu().numpy()
    assert not np.allclose(post, pre, rtol=1e-6)
