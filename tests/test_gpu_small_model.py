"""The drop-in model's float32 layer-body kernels (rk_small_qkv_rope,
rk_small_out_proj, rk_small_logits) against a float64 restatement of the
reference's layer body (engine.py:175-185 RoPE, 244-251 projections, 267
residual, 270-271 logits; pipeline.py:308 first-max argmax)."""

from __future__ import annotations

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2502_15294_b200 import kernels  # noqa: E402


def _rope64(x, pos, freq):
    """engine.py:175-185 in float64: interleaved pairs rotated by pos * freq."""
    ang = pos[:, None, None].astype(np.float64) * freq[None, None, :]
    ev, od = x[..., 0::2], x[..., 1::2]
    out = np.empty_like(x)
    out[..., 0::2] = ev * np.cos(ang) - od * np.sin(ang)
    out[..., 1::2] = ev * np.sin(ang) + od * np.cos(ang)
    return out


@pytest.mark.parametrize("n,dm,heads", [(1, 32, 4), (7, 32, 4), (5, 96, 6), (3, 512, 8), (2, 300, 3)])
def test_small_layer_body_matches_float64(n, dm, heads):
    rng = np.random.default_rng(dm + n)
    x = rng.standard_normal((n, dm)).astype(np.float32)
    w = [(rng.standard_normal((dm, dm)) * dm ** -0.5).astype(np.float32) for _ in range(4)]
    pos = rng.integers(0, 5000, size=n).astype(np.int64)
    dk = dm // heads
    freq = 10000.0 ** (-np.arange(dk // 2, dtype=np.float64) * 2.0 / dk)
    dev = lambda a: torch.from_numpy(a).cuda()  # noqa: E731
    q, k, v = kernels.small_qkv_rope(dev(x), dev(w[0]), dev(w[1]), dev(w[2]), heads, dev(pos), dev(freq))
    x64 = x.astype(np.float64)
    q_ref = _rope64((x64 @ w[0]).reshape(n, heads, dk), pos, freq)
    k_ref = _rope64((x64 @ w[1]).reshape(n, heads, dk), pos, freq).reshape(n, dm)
    v_ref = x64 @ w[2]
    for got, ref in ((q.cpu().numpy(), q_ref), (k.cpu().numpy(), k_ref), (v.cpu().numpy(), v_ref)):
        np.testing.assert_allclose(got, ref, rtol=2e-5, atol=2e-5 * np.abs(ref).max())
    a = rng.standard_normal((n, dm)).astype(np.float32)
    y = kernels.small_out_proj(dev(a), dev(w[3]), dev(x)).cpu().numpy()
    y_ref = x64 + a.astype(np.float64) @ w[3]
    np.testing.assert_allclose(y, y_ref, rtol=2e-5, atol=2e-5 * np.abs(y_ref).max())


@pytest.mark.parametrize("n,dm,vocab", [(1, 32, 258), (4, 64, 258), (3, 128, 1000)])
def test_small_logits_first_max(n, dm, vocab):
    rng = np.random.default_rng(vocab + n)
    x = rng.standard_normal((n, dm)).astype(np.float32)
    emb = rng.standard_normal((vocab, dm)).astype(np.float32)
    emb[vocab // 2] = emb[vocab // 3]          # duplicate rows: ties resolve to the lower index
    x[0] = emb[vocab // 3] * 3.0
    logits, am = kernels.small_logits(torch.from_numpy(x).cuda(), torch.from_numpy(emb).cuda())
    ref = x.astype(np.float64) @ emb.T.astype(np.float64)
    np.testing.assert_allclose(logits.cpu().numpy(), ref, rtol=1e-5, atol=1e-5 * np.abs(ref).max())
    got = am.cpu().numpy()
    lg = logits.cpu().numpy()
    np.testing.assert_array_equal(got, np.argmax(lg, axis=1))   # np.argmax: the first maximum
    assert got[0] == vocab // 3


@pytest.mark.parametrize("n,s,heads,dk,masked", [(5, 40, 4, 8, False), (3, 300, 4, 16, True), (2, 1000, 8, 64, True)])
def test_capture_pre_matches_float64(n, s, heads, dk, masked):
    """capture_mode="pre" (engine.py:187-200): softmax over the visible keys of the
    head-summed logits / (H sqrt(d_k)), float64; a row with no visible key is NaN."""
    rng = np.random.default_rng(s + n)
    q = rng.standard_normal((n, heads, dk)).astype(np.float32)
    k = rng.standard_normal((s, heads * dk)).astype(np.float32)
    q_pos = np.sort(rng.integers(s // 2, s, size=n)).astype(np.int64)
    q_pos[0] = -1 if masked else q_pos[0]                      # row 0 sees nothing when masked
    k_pos = np.arange(s, dtype=np.int64)
    allowed = (rng.random(s) > 0.3) if masked else None
    got = kernels.capture_pre(torch.from_numpy(q).cuda(), torch.from_numpy(k).cuda(), torch.from_numpy(q_pos),
                              torch.from_numpy(k_pos),
                              None if allowed is None else torch.from_numpy(allowed)).cpu().numpy()
    logits = np.einsum("nhd,shd->ns", q.astype(np.float64), k.reshape(s, heads, dk).astype(np.float64))
    logits /= heads * np.sqrt(dk)
    vis = k_pos[None, :] <= q_pos[:, None]
    if allowed is not None:
        vis &= allowed[None, :]
    with np.errstate(invalid="ignore"):
        logits = np.where(vis, logits, -np.inf)
        logits -= logits.max(axis=1, keepdims=True)
        w = np.exp(logits)
        ref = w / w.sum(axis=1, keepdims=True)
    if masked:
        assert np.isnan(got[0]).all() and np.isnan(ref[0]).all()
        got, ref = got[1:], ref[1:]
    np.testing.assert_allclose(got, ref, rtol=1e-12, atol=1e-15)
