"""GPU parity of the tensor-core question prefill (prefill_tc.cu, rk_prefill_attention)
against the oracle: multi-row causal GQA attention over a history + the
question (pipeline.py:225-230, :292-296; kernel contract _attn_ext.pyx:20-81)
and the fused watershed round masses (stats.py:59-94 on the capture of
_attn_ext.pyx:75-76,113-114).  Inputs are bf16-rounded once and fed to both
sides; tolerance 2e-5 relative (north star: 1e-3)."""

from __future__ import annotations

import numpy as np
import pytest

from oracle import attention as oatt
from oracle import rounds as orr

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover - CPU container
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2502_15294_b200 import backend, kernels  # noqa: E402
from paper_2502_15294_b200.errors import DomainError, InvariantError  # noqa: E402
from paper_2502_15294_b200.stats import build_round_items  # noqa: E402

D = 128


def _inputs(rng, n_q, hist, hkv, G, scale=1.0):
    s = hist + n_q
    q = (scale * rng.standard_normal((n_q, hkv * G, D))).astype(np.float32)
    k = oatt.round_to_bf16(rng.standard_normal((s, hkv, D)).astype(np.float32))
    v = oatt.round_to_bf16(rng.standard_normal((s, hkv, D)).astype(np.float32))
    qp = np.arange(hist, s)
    kp = np.arange(s)
    return q, k, v, qp, kp


def _dev(q, k, v, qp, kp, allowed=None):
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()  # noqa: E731
    al = None if allowed is None else t(allowed.astype(np.uint8))
    return t(q), t(k).bfloat16(), t(v).bfloat16(), t(qp.astype(np.int64)), t(kp.astype(np.int64)), al


def _rel(got, ref):
    return float(np.abs(got - ref).max() / np.abs(ref).max())


@pytest.mark.parametrize("n_q,hist,hkv,G", [
    (16, 1000, 2, 4),       # 64 stacked rows: one M tile per kv-head
    (100, 2500, 2, 7),      # Qwen2-style group, ragged tiles
    (200, 777, 1, 1),       # MHA, 2 M tiles, history not a multiple of 64
    (64, 0, 4, 4),          # question only (pure causal)
    (513, 4096, 4, 7),      # C3-like question length, several chunks per M tile
])
def test_prefill_vs_oracle(rng, n_q, hist, hkv, G):
    q, k, v, qp, kp = _inputs(rng, n_q, hist, hkv, G, scale=2.0)
    ref, _ = oatt.attention_forward_gqa(q, k, v, qp, kp)
    tq, tk, tv, tqp, tkp, _ = _dev(q, k, v, qp, kp)
    out, raw, bad = kernels.prefill_attention(tq, tk, tv, tqp, tkp)
    torch.cuda.synchronize()
    assert raw is None and int(bad.item()) == 2**31 - 1
    err = _rel(out.reshape(n_q, -1).cpu().numpy(), ref)
    assert err < 2e-5, err


def test_prefill_peaked_attention(rng):
    """Sharp softmax (logits ~ +-40 in log2 units) exercises the lazy rescale and
    the P split.  The q = q_hi + q_lo split carries 16 mantissa bits, so the
    logit error grows with |logit|: ~3e-5 relative here (north star: 1e-3)."""
    q, k, v, qp, kp = _inputs(rng, 96, 1500, 2, 4, scale=12.0)
    ref, _ = oatt.attention_forward_gqa(q, k, v, qp, kp)
    out, _, _ = kernels.prefill_attention(*_dev(q, k, v, qp, kp)[:5])
    err = _rel(out.reshape(96, -1).cpu().numpy(), ref)
    assert err < 1e-4, err


def test_prefill_allowed_mask_and_positions(rng):
    """`allowed` mask (mask mode, pipeline.py:271-280) and non-contiguous positions."""
    n_q, hist, hkv, G = 40, 1200, 2, 4
    q, k, v, qp, kp = _inputs(rng, n_q, hist, hkv, G)
    kp = kp * 3 + 5                     # gaps in the positions
    qp = kp[hist:].copy()
    allowed = rng.random(hist + n_q) < 0.6
    allowed[hist:] = True
    ref, _ = oatt.attention_forward_gqa(q, k, v, qp, kp, allowed=allowed)
    out, _, _ = kernels.prefill_attention(*_dev(q, k, v, qp, kp)[:5],
                                          allowed=_dev(q, k, v, qp, kp, allowed)[5])
    assert _rel(out.reshape(n_q, -1).cpu().numpy(), ref) < 2e-5


def test_prefill_no_visible_key_reports_row(rng):
    q, k, v, qp, kp = _inputs(rng, 32, 100, 2, 4)
    qp = qp.copy()
    qp[7] = -1                          # row 7 sees nothing
    out, _, bad = kernels.prefill_attention(*_dev(q, k, v, qp, kp)[:5])
    assert int(bad.item()) == 7


@pytest.mark.parametrize("n_q,G,hkv,n_rounds", [(64, 4, 2, 9), (200, 7, 4, 12), (512, 7, 4, 16)])
def test_prefill_fused_scoring_vs_oracle(rng, n_q, G, hkv, n_rounds):
    """Output AND Eq. 1 masses from one pass equal attention_forward(capture) +
    aggregate_round_attention (pipeline.py:225-245)."""
    lens = rng.integers(100, 700, size=n_rounds)
    starts = np.concatenate([[0], np.cumsum(lens)])
    hist = int(starts[-1])
    q, k, v, qp, kp = _inputs(rng, n_q, hist, hkv, G, scale=1.5)
    s = hist + n_q
    ref_out, cap = oatt.attention_forward_gqa(q, k, v, qp, kp, capture=True)
    rounds = [orr.Round(m, (int(starts[m]), int(starts[m]) + 5), (int(starts[m]) + 5, int(starts[m + 1])))
              for m in range(n_rounds)]
    rounds.append(orr.Round(n_rounds, (hist, s), (s, s)))
    active = [m for m in range(n_rounds) if m != 3]
    ref_raw = orr.aggregate_round_attention(cap, rounds, "question", n_rounds, active_rounds=active,
                                            row_offset=hist)
    bounds = [(int(starts[m]), int(starts[m + 1]), m) for m in range(n_rounds)] + [(hist, s, n_rounds)]
    items = torch.from_numpy(build_round_items(bounds, 1024)).cuda()
    act = torch.tensor([m in active for m in range(n_rounds)], dtype=torch.uint8, device="cuda")
    out, raw, _ = kernels.prefill_attention(*_dev(q, k, v, qp, kp)[:5], items=items, n_bins=n_rounds, active=act)
    assert _rel(out.reshape(n_q, -1).cpu().numpy(), ref_out) < 2e-5
    np.testing.assert_allclose(raw.cpu().numpy(), ref_raw, rtol=2e-5, atol=1e-9)
    # the selection made from these masses is the reference's
    pol = orr.SelectionPolicy("top_percent", fraction=0.25)
    assert orr.select(orr.normalize(raw.cpu().numpy()), pol) == orr.select(orr.normalize(ref_raw), pol)


def test_kernel_contract_routes_multirow_bf16_to_tensor_cores(rng, monkeypatch):
    """backend.attention_forward_gqa on >= 64 stacked bf16 rows (tcgen05 path)
    matches the oracle, capture included, and equals the CUDA-core split kernel."""
    n_q, hist, hkv, G = 48, 900, 2, 4
    q, k, v, qp, kp = _inputs(rng, n_q, hist, hkv, G)
    ref_out, ref_sc = oatt.attention_forward_gqa(q, k, v, qp, kp, capture=True)
    tq, tk, tv, tqp, tkp, _ = _dev(q, k, v, qp, kp)
    out, sc = backend.attention_forward_gqa(tq, tk, tv, tqp, tkp, capture=True)
    np.testing.assert_allclose(out.cpu().numpy(), ref_out, rtol=1e-4, atol=2e-5)
    np.testing.assert_allclose(sc.cpu().numpy(), ref_sc, rtol=1e-4, atol=1e-8)
    with pytest.raises(InvariantError):
        backend.attention_forward_gqa(tq, tk, tv, tqp - 10**6, tkp)


def test_prefill_single_pass_bf16_path(rng):
    """RK_PREFILL_SINGLE_PASS: q and P rounded to bf16, one MMA pass each (the
    bf16 path, stated separately from the fp32-class default): max error within
    3e-2 of the output range, mean within 3e-3; scoring is refused on it."""
    n_q, hist, hkv, G = 200, 3000, 2, 7
    q, k, v, qp, kp = _inputs(rng, n_q, hist, hkv, G, scale=1.0)
    ref, _ = oatt.attention_forward_gqa(q, k, v, qp, kp)
    args = _dev(q, k, v, qp, kp)[:5]
    out, _, _ = kernels.prefill_attention(*args, single_pass=True)
    got = out.reshape(n_q, -1).cpu().numpy()
    assert _rel(got, ref) < 3e-2
    assert float(np.abs(got - ref).mean() / np.abs(ref).max()) < 3e-3
    items = torch.from_numpy(build_round_items([(0, hist, 0), (hist, hist + n_q, 1)], 1024)).cuda()
    with pytest.raises(DomainError):
        kernels.prefill_attention(*args, items=items, n_bins=1, single_pass=True)


def test_prefill_randomized_shapes_vs_oracle():
    """Seeded sweep of question rows, history, kv-heads and groups (>= 64 stacked
    rows), with the fused round masses on half of them: outputs vs the oracle
    (2e-5) and masses vs capture + aggregate (2e-5) through the balanced planner."""
    rng = np.random.default_rng(77)
    for i in range(10):
        hkv = int(rng.choice([1, 2, 4, 8]))
        G = int(rng.choice([1, 2, 4, 7, 8]))
        n_q = int(rng.integers(max(1, -(-64 // G)), 300))
        n_r = int(rng.integers(1, 9))
        lens = rng.integers(1, 600, size=n_r)
        starts = np.concatenate([[0], np.cumsum(lens)])
        hist = int(starts[-1])
        q, k, v, qp, kp = _inputs(rng, n_q, hist, hkv, G, scale=1.5)
        s = hist + n_q
        ref, cap = oatt.attention_forward_gqa(q, k, v, qp, kp, capture=True)
        args = _dev(q, k, v, qp, kp)[:5]
        if i % 2:
            bounds = [(int(starts[m]), int(starts[m + 1]), m) for m in range(n_r)] + [(hist, s, n_r)]
            items = torch.from_numpy(build_round_items(bounds, 1024)).cuda()
            out, raw, _ = kernels.prefill_attention(*args, items=items, n_bins=n_r)
            rounds = [orr.Round(m, (int(starts[m]), int(starts[m]) + 1), (int(starts[m]) + 1, int(starts[m + 1])))
                      for m in range(n_r)]
            rounds.append(orr.Round(n_r, (hist, s), (s, s)))
            ref_raw = orr.aggregate_round_attention(cap, rounds, "question", n_r, row_offset=hist)
            np.testing.assert_allclose(raw.cpu().numpy(), ref_raw, rtol=2e-5, atol=1e-9)
        else:
            out, _, _ = kernels.prefill_attention(*args)
        err = _rel(out.reshape(n_q, -1).cpu().numpy(), ref)
        assert err < 2e-5, (i, n_q, hist, hkv, G, err)
