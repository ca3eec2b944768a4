"""GPU parity of the tcgen05 projection kernels (csrc/proj.cu) — the decode
step's layer body, engine.py:244-251,267-271 of the reference: q, k =
RoPE(x W_q), RoPE(x W_k); v = x W_v; x += out W_o; logits = x E^T + first
argmax — against a float64 restatement on the same bf16 weights, across row
counts (1 .. 100: the 16 / 32 / 64-column tiles and the 64-row launch split),
Llama-3-8B / Qwen2-7B / toy shapes (split-K over many CTAs and one CTA per
strip group), plus determinism and the self-resetting split-K tickets."""

from __future__ import annotations

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2502_15294_b200 import _lib, kernels  # noqa: E402
from paper_2502_15294_b200.decode_model import rope_freq  # noqa: E402


def _rope64(y, pos, d, freq):
    """engine.py:175-185: interleaved pairs, float64 angles."""
    m, width = y.shape
    out = y.copy()
    i = (np.arange(width) % d) // 2
    ang = pos[:, None].astype(np.float64) * freq[i][None, :]
    c, s = np.cos(ang), np.sin(ang)
    x0, x1 = y[:, 0::2], y[:, 1::2]
    out[:, 0::2] = x0 * c[:, 0::2] - x1 * s[:, 0::2]
    out[:, 1::2] = x0 * s[:, 1::2] + x1 * c[:, 1::2]
    return out


SHAPES = [(32, 8, 128), (28, 4, 128), (8, 8, 64), (8, 2, 128)]


@pytest.mark.parametrize("mode", ["cluster", "ticket"])
@pytest.mark.parametrize("hq,hkv,d", SHAPES)
@pytest.mark.parametrize("m", [1, 3, 16, 17, 32, 40, 64, 100])
def test_qkv_rope_matches_float64(hq, hkv, d, m, mode, monkeypatch):
    if mode == "ticket":
        monkeypatch.setenv("RK_PROJ_NO_CLUSTER", "1")
    g = torch.Generator(device="cuda").manual_seed(1000 * m + hq)
    D = hq * d
    qd, kd = hq * d, hkv * d
    w = (torch.randn((D, qd + 2 * kd), generator=g, device="cuda") / np.sqrt(D)).to(torch.bfloat16)
    x = torch.randn((m, D), generator=g, device="cuda")
    pos = torch.randint(0, 200000, (m,), generator=g, device="cuda", dtype=torch.int32)
    freq = torch.from_numpy(rope_freq(d, 10000.0)).cuda()
    q = torch.full((m, hq, d), float("nan"), device="cuda")
    stride = 3 * kd                                        # cache rows wider than one row (strided append)
    kbuf = torch.zeros((m, stride), dtype=torch.bfloat16, device="cuda")
    vbuf = torch.zeros((m, stride), dtype=torch.bfloat16, device="cuda")
    wp = kernels.pack_weight(w)
    ws = kernels.proj_workspace(m, D, qd + 2 * kd, "cuda")
    kernels.qkv_rope(x, wp, hq, hkv, d, pos, freq, q, kbuf, vbuf, kv_row_stride=stride, ws=ws)
    torch.cuda.synchronize()
    y = x.double().cpu().numpy() @ w.double().cpu().numpy()
    ref = _rope64(y[:, :qd + kd], pos.cpu().numpy(), d, rope_freq(d, 10000.0))
    scale = np.abs(ref).max()
    err_q = np.abs(q.view(m, -1).double().cpu().numpy() - ref[:, :qd]).max() / scale
    assert err_q < 1e-5, err_q
    # k / v rows: bf16 of the fp32-class values (one bf16 ulp at most)
    kg = kbuf[:, :kd].double().cpu().numpy()
    vg = vbuf[:, :kd].double().cpu().numpy()
    assert np.all(np.abs(kg - ref[:, qd:]) <= 2 ** -7 * np.abs(ref[:, qd:]) + 1e-5 * scale)
    assert np.all(np.abs(vg - y[:, qd + kd:]) <= 2 ** -7 * np.abs(y[:, qd + kd:]) + 1e-5 * scale)
    assert int(ws[:4096].count_nonzero()) == 0            # split-K tickets back at zero
    assert torch.all(kbuf[:, kd:] == 0) and torch.all(vbuf[:, kd:] == 0)


@pytest.mark.parametrize("mode", ["cluster", "ticket"])
@pytest.mark.parametrize("k,n", [(4096, 4096), (3584, 3584), (512, 512), (4096, 384)])
@pytest.mark.parametrize("m", [1, 16, 33, 64, 70])
def test_out_proj_accumulates_residual(k, n, m, mode, monkeypatch):
    """Both split-K reductions: partials added through distributed shared memory
    inside a cluster per strip group, or published and added by the last CTA
    of a ticket (RK_PROJ_NO_CLUSTER)."""
    if mode == "ticket":
        monkeypatch.setenv("RK_PROJ_NO_CLUSTER", "1")
    g = torch.Generator(device="cuda").manual_seed(7 * m + k)
    w = (torch.randn((k, n), generator=g, device="cuda") / np.sqrt(k)).to(torch.bfloat16)
    a = torch.randn((m, k), generator=g, device="cuda")
    resid = torch.randn((m, n), generator=g, device="cuda")
    r0 = resid.double().cpu().numpy()
    kernels.out_proj(a, kernels.pack_weight(w), resid)
    torch.cuda.synchronize()
    ref = r0 + a.double().cpu().numpy() @ w.double().cpu().numpy()
    err = np.abs(resid.double().cpu().numpy() - ref).max() / np.abs(ref).max()
    assert err < 1e-5, err


@pytest.mark.parametrize("mode", ["cluster", "ticket"])
def test_projection_deterministic(mode, monkeypatch):
    """Split-K partials are added in CTA order: repeated launches are bitwise equal."""
    if mode == "ticket":
        monkeypatch.setenv("RK_PROJ_NO_CLUSTER", "1")
    g = torch.Generator(device="cuda").manual_seed(3)
    w = (torch.randn((4096, 4096), generator=g, device="cuda") / 64).to(torch.bfloat16)
    wp = kernels.pack_weight(w)
    a = torch.randn((16, 4096), generator=g, device="cuda")
    outs = []
    for _ in range(4):
        r = torch.zeros((16, 4096), device="cuda")
        kernels.out_proj(a, wp, r)
        outs.append(r)
    torch.cuda.synchronize()
    for o in outs[1:]:
        assert torch.equal(o, outs[0])


@pytest.mark.parametrize("m", [1, 5, 32, 64, 130])       # 130: three 64-row launches (B=256 groups of 128)
def test_lm_head_first_argmax(m):
    """Tied logits + first argmax (np.argmax) + next-token embedding; ties
    planted between two vocabulary rows go to the lower id."""
    V, D = 258, 512
    g = torch.Generator(device="cuda").manual_seed(m)
    emb = torch.randn((V, D), generator=g, device="cuda").to(torch.bfloat16)
    emb[200] = emb[17]                                  # identical rows: exact logit ties
    x = torch.randn((m, D), generator=g, device="cuda")
    x[0] = emb[17].float() * 3.0                          # row 0's maximum is the 17 / 200 tie
    xn = torch.zeros_like(x)
    tokens = torch.zeros(m, dtype=torch.int32, device="cuda")
    pos = torch.arange(m, dtype=torch.int32, device="cuda")
    kernels.lm_head(x, kernels.pack_weight(emb.t().contiguous()), V, emb, xn, tokens, pos)
    torch.cuda.synchronize()
    logits = x.double().cpu().numpy() @ emb.double().cpu().numpy().T
    want = logits.argmax(axis=1)
    got = tokens.cpu().numpy()
    assert got[0] == 17
    # a flip needs a near-tie below the fp32-class error
    srt = np.sort(logits, axis=1)
    for i in range(m):
        if got[i] != want[i]:
            assert srt[i, -1] - srt[i, -2] < 1e-5 * np.abs(srt[i, -1]), i
    np.testing.assert_array_equal(xn.cpu().numpy(), emb[tokens.long()].float().cpu().numpy())
    np.testing.assert_array_equal(pos.cpu().numpy(), np.arange(m) + 1)


def test_projection_workspace_capacity_error():
    w = kernels.pack_weight(torch.zeros((512, 512), dtype=torch.bfloat16, device="cuda"))
    a = torch.zeros((16, 512), device="cuda")
    r = torch.zeros((16, 512), device="cuda")
    small = torch.zeros(256, dtype=torch.uint8, device="cuda")
    with pytest.raises(Exception, match="workspace"):
        _lib.call("rk_out_proj", _lib.ptr(a), 16, 512, _lib.ptr(w), 512, _lib.ptr(r), _lib.ptr(small), 256,
                  _lib.stream_ptr(None))
