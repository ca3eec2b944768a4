"""GPU parity of the small-batch cluster decode (decode_cluster.cu: one
thread-block cluster per (dialogue, kv-head), split-K merged in distributed
shared memory) against the oracle — the decode loop's attention,
pipeline.py:298-313 -> engine.py:244-267 with one row (kernel contract
_attn_ext.pyx:20-81) — over every cluster size the planner picks (16/8/4/2/1),
ragged and tiny lengths, d 64/128 and all supported groups; plus the
persistent split-K kernel at the same small shapes with the cluster path
disabled (RK_DECODE_CLUSTER=0, read once per process -> subprocess)."""

from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

from oracle import attention as oatt

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2502_15294_b200 import kernels  # noqa: E402

ROOT = Path(__file__).resolve().parents[1]


def _run(lens, hkv, G, d, append=True, cap=None, seed=0, dtype=None):
    dtype = dtype or torch.bfloat16
    B = len(lens)
    lens = np.array(lens)
    cap = cap or int(lens.max()) + 1
    g = torch.Generator(device="cuda").manual_seed(seed)
    kc = torch.randn(B, cap, hkv, d, device="cuda", generator=g).to(dtype)
    vc = torch.randn(B, cap, hkv, d, device="cuda", generator=g).to(dtype)
    q = 2.0 * torch.randn(B, hkv * G, d, device="cuda", generator=g)
    kn = torch.randn(B, hkv, d, device="cuda", generator=g).to(dtype) if append else None
    vn = torch.randn(B, hkv, d, device="cuda", generator=g).to(dtype) if append else None
    sl = torch.from_numpy(lens.astype(np.int32)).cuda()
    max_len = int(lens.max()) + (1 if append else 0)
    plan = kernels.decode_plan(B, hkv * G, hkv, d, dtype, max_len, kc.stride(0))
    out = kernels.decode_attention(q, kc, vc, sl, max_len, k_new=kn, v_new=vn)
    torch.cuda.synchronize()
    worst = 0.0
    for b in range(B):
        L = int(lens[b]) + (1 if append else 0)
        kk = kc[b, :L].float().cpu().numpy()
        vv = vc[b, :L].float().cpu().numpy()
        if append:       # the appended row landed in the cache
            np.testing.assert_array_equal(kk[L - 1], kn[b].float().cpu().numpy())
            np.testing.assert_array_equal(vv[L - 1], vn[b].float().cpu().numpy())
        ref, _ = oatt.attention_forward_gqa(q[b:b + 1].cpu().numpy(), kk, vv, [L - 1], np.arange(L))
        err = np.abs(out[b].reshape(1, -1).cpu().numpy() - ref).max() / np.abs(ref).max()
        worst = max(worst, float(err))
    return plan, worst


@pytest.mark.parametrize("lens,hkv,G,d", [
    ([16512], 8, 4, 128),                 # B=1 C2 lower layer
    ([2176], 8, 4, 128),                  # B=1 C2 upper layer (kept rounds)
    ([3000, 1100], 8, 4, 128),            # B=2, ragged
    ([700, 2999, 64, 1500], 8, 4, 128),   # B=4, ragged, one dialogue shorter than a stage
    ([2999] * 8, 8, 4, 128),              # C=2
    ([2999, 17, 1024, 1, 700, 2048, 5, 333, 1500, 64, 2999, 900], 8, 4, 128),   # C=1, ragged/tiny
    ([5000], 4, 7, 128),                  # Qwen2-style group (C3 shape): 4 clusters of 16
    ([4000, 333], 2, 8, 64),              # d=64, G=8
    ([1234], 8, 1, 128),                  # MHA
    ([900, 901, 902], 4, 2, 64),
])
def test_cluster_decode_vs_oracle(lens, hkv, G, d):
    """The cluster size depends on how many clusters the GPCs hold at once
    (B200: 7 of 16, 15 of 8, ...): checked as a plan property, not a constant."""
    plan, err = _run(lens, hkv, G, d)
    pairs = len(lens) * hkv
    assert plan > 0 and pairs * plan <= torch.cuda.get_device_properties(0).multi_processor_count, plan
    if pairs * 2 > 148:
        assert plan == 1
    assert err < 2e-5, (plan, err)      # north star: 1e-3 relative


def test_cluster_decode_without_append_and_slack_capacity():
    """No appended row; the cache capacity exceeds the lengths (the TMA map
    spans the capacity, slices stop at each dialogue's length)."""
    plan, err = _run([1000, 2500, 40], 8, 4, 128, append=False, cap=4096)
    assert plan > 1 and err < 2e-5


def test_cluster_decode_single_key():
    """A dialogue whose only key is the appended one (len 0 + 1)."""
    plan, err = _run([0, 3000], 8, 4, 128)
    assert plan > 0 and err < 2e-5


def test_cluster_decode_in_cuda_graph_repeats():
    """Replayed from a CUDA graph (the engine's capture) with PDL between
    calls: identical outputs on every replay, equal to the eager call."""
    B, hkv, G, d, S = 2, 8, 4, 128, 2500
    kc = torch.randn(B, S + 1, hkv, d, device="cuda").bfloat16()
    vc = torch.randn(B, S + 1, hkv, d, device="cuda").bfloat16()
    q = torch.randn(B, hkv * G, d, device="cuda")
    sl = torch.full((B,), S, dtype=torch.int32, device="cuda")
    kn = torch.randn(B, hkv, d, device="cuda").bfloat16()
    vn = torch.randn(B, hkv, d, device="cuda").bfloat16()
    outs = [torch.empty(B, hkv * G, d, device="cuda") for _ in range(4)]
    st = torch.cuda.Stream()
    st.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(st):
        ref = kernels.decode_attention(q, kc, vc, sl, S + 1, k_new=kn, v_new=vn).clone()
        gr = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gr, stream=st):
            for o in outs:
                kernels.decode_attention(q, kc, vc, sl, S + 1, k_new=kn, v_new=vn, out=o)
        for _ in range(3):
            gr.replay()
    torch.cuda.synchronize()
    for o in outs:
        assert torch.equal(o, ref)


def test_persistent_split_k_at_small_batches_subprocess():
    """RK_DECODE_CLUSTER=0: the persistent split-K + merge kernel serves the
    same small shapes (plan 0) and matches the oracle."""
    code = (
        "import sys; sys.path.insert(0, %r); sys.path.insert(0, %r)\n"
        "from test_gpu_decode_cluster import _run\n"
        "for lens in ([2176], [3000, 1100], [2999, 17, 1024, 1]):\n"
        "    plan, err = _run(lens, 8, 4, 128)\n"
        "    assert plan == 0, plan\n"
        "    assert err < 2e-5, err\n"
        "print('ok')\n" % (str(ROOT), str(ROOT / "tests")))
    env = dict(os.environ, RK_DECODE_CLUSTER="0")
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0 and r.stdout.strip().endswith("ok"), r.stdout + r.stderr


def test_cluster_decode_on_engine_layer_views_at_capacity():
    """Caches as the engine holds them: layer l's K / V are strided views of one
    [B][L][2][S][Hkv][d] tensor (dialogue stride = L*2*S rows), every dialogue
    filled to capacity by the appended row — the last view ends at the end of
    the allocation, so no tail box may read past it."""
    B, L, S, hkv, G, d = 4, 3, 1500, 4, 7, 128
    big = torch.randn(B, L, 2, S, hkv, d, device="cuda").bfloat16()
    q = torch.randn(B, hkv * G, d, device="cuda")
    kn = torch.randn(B, hkv, d, device="cuda").bfloat16()
    vn = torch.randn(B, hkv, d, device="cuda").bfloat16()
    for layer in range(L):
        kc, vc = big[:, layer, 0], big[:, layer, 1]
        sl = torch.tensor([S - 1, S - 700, S - 1, S - 30], dtype=torch.int32, device="cuda")
        assert kernels.decode_plan(B, hkv * G, hkv, d, torch.bfloat16, S, kc.stride(0)) > 0
        out = kernels.decode_attention(q, kc, vc, sl, S, k_new=kn, v_new=vn)
        torch.cuda.synchronize()
        for b in range(B):
            n = int(sl[b]) + 1
            kk = kc[b, :n].float().cpu().numpy()
            vv = vc[b, :n].float().cpu().numpy()
            ref, _ = oatt.attention_forward_gqa(q[b:b + 1].cpu().numpy(), kk, vv, [n - 1], np.arange(n))
            err = np.abs(out[b].reshape(1, -1).cpu().numpy() - ref).max() / np.abs(ref).max()
            assert err < 2e-5, (layer, b, err)


def test_randomized_shapes_vs_oracle():
    """Seeded sweep over batch (1-18), kv-heads, group, head dim, ragged lengths
    and append on/off: every shape goes through rk_decode_attention's planner
    (cluster sizes 1-16, or the persistent kernel) and matches the oracle."""
    rng = np.random.default_rng(2024)
    plans = set()
    for i in range(24):
        hkv = int(rng.choice([2, 4, 8]))
        G = int(rng.choice([1, 2, 4, 7, 8]))
        d = int(rng.choice([64, 128]))
        B = int(rng.integers(1, 19))
        lens = [int(x) for x in rng.integers(0, 4000, size=B)]
        if rng.random() < 0.5:
            lens = [max(lens)] * B                     # equal lengths (the engine's batches)
        append = bool(rng.random() < 0.8)
        if not append:
            lens = [max(1, x) for x in lens]
        plan, err = _run(lens, hkv, G, d, append=append, seed=100 + i)
        plans.add(plan)
        assert err < 2e-5, (i, B, hkv, G, d, append, plan, err)
    assert any(p > 1 for p in plans) and any(p >= 0 for p in plans), plans


@pytest.mark.parametrize("lens,hkv,G,d", [
    ([16512], 8, 4, 128),                 # B=1 C2 lower layer, fp32 KV (the reference's precision)
    ([2176], 8, 4, 128),
    ([3000, 1100], 8, 4, 128),
    ([700, 2999, 64, 1500], 8, 4, 128),   # ragged, one dialogue shorter than a stage
    ([2999] * 8, 8, 4, 128),
    ([2999, 17, 1024, 1, 700, 2048, 5, 333, 1500, 64, 2999, 900], 8, 4, 128),
    ([5000], 4, 7, 128),
    ([4000, 333], 2, 8, 64),
    ([1234], 8, 1, 128),
    ([63, 64, 65, 127, 129], 4, 2, 64),   # stage (64 keys) boundaries
])
def test_cluster_decode_f32_vs_oracle(lens, hkv, G, d):
    """fp32 KV on the cluster decode (64-key fp32 stages, two alternating consumer
    warp sets, K / V split into bf16 hi + lo on the fly): outputs within 2e-5
    relative of the fp64 oracle on the identical fp32 inputs (_attn_np.py:26-28)."""
    plan, err = _run(lens, hkv, G, d, dtype=torch.float32, seed=3)
    assert plan > 0, plan
    assert err < 2e-5, err         # same class as the bf16 path; north star: 1e-3
