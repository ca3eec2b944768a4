"""The serving engine's model: the reference's toy transformer (engine.py:146-287 —
attention + residual only, RoPE, tied logits, byte vocabulary of 258) at the
BASELINE configurations' shapes (Llama-3-8B: 32 layers, 32 query / 8 key-value
heads of 128; Qwen2-7B: 28 layers, 28 / 4), with GQA projections (W_k, W_v:
d_model x Hkv*d — the reference is MHA only) and bf16 weights.

Weights are random-initialised like the reference (engine.py:152-161: N(0,1)
embedding; W_q, W_k, W_v ~ N(0,1)/sqrt(d_model); W_o additionally / sqrt(2L)),
drawn on the device, and packed once into the tensor-core fragment order of the
decode projections (rk_pack_weight).  Tests may pass explicit weights.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import kernels

VOCAB_SIZE = 258        # 256 bytes + SEP + EOT (conversation.py:23-26)
SEP_TOKEN = 256
EOT_TOKEN = 257


@dataclass(frozen=True)
class ModelShape:
    num_layers: int = 32
    hq: int = 32
    hkv: int = 8
    head_dim: int = 128
    vocab: int = VOCAB_SIZE
    rope_theta: float = 10000.0

    @property
    def d_model(self) -> int:
        return self.hq * self.head_dim

    @property
    def qkv_width(self) -> int:
        return (self.hq + 2 * self.hkv) * self.head_dim


def rope_freq(head_dim: int, theta: float) -> np.ndarray:
    """The reference's RoPE frequencies, engine.py:162-164 (float64)."""
    half = head_dim // 2
    return theta ** (-np.arange(half, dtype=np.float64) * 2.0 / head_dim)


class DecodeModel:
    """bf16 weights in two forms: packed for the fused decode projections
    (rk_qkv_rope / rk_out_proj / rk_lm_head) and, when `prefill_gemm`, plain
    row-major for the multi-row question prefill's library GEMMs."""

    def __init__(self, shape: ModelShape, device="cuda", seed: int = 42, weights: dict | None = None,
                 prefill_gemm: bool = False, shard: tuple[int, int] = (0, 1)):
        """shard = (rank, world): KV-head sharding of every dialogue over `world`
        ranks (SURVEY §8e's option for fewer dialogues than GPUs).  The same
        seeded weights are drawn; this rank keeps the columns of W_q / W_k / W_v
        of its query heads [rank hq/world, ...) and kv-heads [rank hkv/world, ...)
        and the matching rows of W_o (a row-parallel output projection whose
        partial sums the engine all-reduces); the tied embedding stays whole."""
        self.shape = s = shape
        self.device = dev = torch.device(device)
        D, L = s.d_model, s.num_layers
        rank, world = shard
        if world < 1 or not 0 <= rank < world or s.hkv % world:
            raise ValueError(f"shard {shard}: kv-heads {s.hkv} must split evenly over the ranks")
        self.shard = (rank, world)
        self.hq_local, self.hkv_local = s.hq // world, s.hkv // world
        qs = slice(rank * self.hq_local * s.head_dim, (rank + 1) * self.hq_local * s.head_dim)
        ks = slice(rank * self.hkv_local * s.head_dim, (rank + 1) * self.hkv_local * s.head_dim)
        self.freq = torch.from_numpy(rope_freq(s.head_dim, s.rope_theta)).to(dev)
        self.w_qkv_packed, self.w_o_packed = [], []
        self.w_qkv_kn, self.w_o_kn = [], []
        if weights is None:
            g = torch.Generator(device=dev).manual_seed(seed)
            scale = D ** -0.5
            emb = torch.randn((s.vocab, D), generator=g, device=dev)
        else:
            emb = torch.as_tensor(weights["emb"], dtype=torch.float32).to(dev)
        self.emb = emb.to(torch.bfloat16).contiguous()               # [V][D] lookup table (tied)
        self.emb_packed = kernels.pack_weight(self.emb.t().contiguous())   # logits = x @ E^T
        for l in range(L):
            if weights is None:
                wq = torch.randn((D, s.hq * s.head_dim), generator=g, device=dev) * scale
                wk = torch.randn((D, s.hkv * s.head_dim), generator=g, device=dev) * scale
                wv = torch.randn((D, s.hkv * s.head_dim), generator=g, device=dev) * scale
                wo = torch.randn((s.hq * s.head_dim, D), generator=g, device=dev) * (scale / np.sqrt(2.0 * L))
            else:
                wq, wk, wv, wo = (torch.as_tensor(weights[n][l], dtype=torch.float32).to(dev)
                                  for n in ("wq", "wk", "wv", "wo"))
            wqkv = torch.cat([wq[:, qs], wk[:, ks], wv[:, ks]], dim=1).to(torch.bfloat16).contiguous()
            wo16 = wo[qs].to(torch.bfloat16).contiguous()               # (hq_local d, D)
            self.w_qkv_packed.append(kernels.pack_weight(wqkv))
            self.w_o_packed.append(kernels.pack_weight(wo16))
            if prefill_gemm:
                self.w_qkv_kn.append(wqkv)
                self.w_o_kn.append(wo16)
            del wq, wk, wv, wo, wqkv, wo16
        torch.cuda.synchronize(dev)

    def weight_bytes_per_token(self) -> int:
        """Algorithmic weight bytes of one decode token step (bf16 W_q|W_k|W_v
        and W_o of every layer + the tied embedding; the 128-row padding of the
        stored logits operand is not counted)."""
        s = self.shape
        qkv_w = (self.hq_local + 2 * self.hkv_local) * s.head_dim
        o_rows = self.hq_local * s.head_dim
        return 2 * (s.num_layers * (s.d_model * qkv_w + o_rows * s.d_model) + s.vocab * s.d_model)

    def host_weights(self) -> dict:
        """The bf16 weights as float32 NumPy (for the oracle)."""
        s = self.shape
        if self.shard[1] > 1:
            raise ValueError("host_weights of a head-sharded model: use the unsharded model")
        qd, kd = s.hq * s.head_dim, s.hkv * s.head_dim
        out = {"emb": self.emb.float().cpu().numpy(), "wq": [], "wk": [], "wv": [], "wo": []}
        if not self.w_qkv_kn:
            raise ValueError("host_weights needs prefill_gemm=True (row-major copies)")
        for l in range(s.num_layers):
            w = self.w_qkv_kn[l].float().cpu().numpy()
            out["wq"].append(w[:, :qd])
            out["wk"].append(w[:, qd:qd + kd])
            out["wv"].append(w[:, qd + kd:])
            out["wo"].append(self.w_o_kn[l].float().cpu().numpy())
        return out
