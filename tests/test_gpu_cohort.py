"""Cohort serving (cohort.py): two phase-offset cohorts share one decode loop
with row masks; every dialogue's kept rounds and answer ids must equal a plain
single-group engine's over the same turns (the row-masked kernels touch only the
active rows, and every row's arithmetic is independent of the others)."""

from __future__ import annotations

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2502_15294_b200 import kernels  # noqa: E402
from paper_2502_15294_b200.cohort import CohortDecoder  # noqa: E402
from paper_2502_15294_b200.decode_engine import EngineConfig, RoundDecodeEngine  # noqa: E402
from paper_2502_15294_b200.decode_model import DecodeModel  # noqa: E402
from paper_2502_15294_b200.selection import SelectionPolicy  # noqa: E402


def _cfg(**kw):
    base = dict(num_layers=4, watershed=2, hq=8, hkv=2, head_dim=128, rounds=7, round_tokens=64, batch=4,
                decode_steps=6, policy=SelectionPolicy("top_percent", fraction=0.3), item_chunk=32, plant=2,
                plant_beta=0.3, question_variants=2, model_seed=5)
    base.update(kw)
    return EngineConfig(**base)


@pytest.mark.parametrize("turns,cohorts,rows", [(1, 2, 1), (3, 2, 1), (3, 4, 1), (2, 2, 24)])
def test_cohorts_match_single_group(turns, cohorts, rows):
    """rows > 1: multi-row questions (tcgen05 prefill prologue, fused scoring)."""
    cfg = _cfg(question_rows=rows)
    dialogues = [2, 5, 9, 11]
    co = CohortDecoder(cfg, cohorts=cohorts, dialogues=dialogues)
    co.prepare()
    co.run_turns(turns)
    kept = co.last_kept_by_dialogue
    got = co.answers()
    ref = RoundDecodeEngine(cfg, model=DecodeModel(cfg.shape, "cuda", seed=cfg.model_seed, prefill_gemm=rows > 1),
                            dialogues=dialogues)
    ref.prepare()
    # prepare ran one eager turn on both sides (each cohort engine and the reference)
    for _ in range(turns):
        k_ref, _ = ref.run_turn()
    torch.cuda.synchronize()
    want = ref.answers()
    for b, gid in enumerate(dialogues):
        assert kept[gid] == [int(x) for x in k_ref[b]], (gid, kept[gid], k_ref[b])
        np.testing.assert_array_equal(got[b], want[b])


def test_row_masked_kernels_leave_inactive_rows():
    """rk_decode_attention_rows / rk_out_proj_rows / rk_lm_head_rows: inactive rows
    get no append, no length advance, no residual update, no token."""
    B, hkv, G, d, S = 4, 8, 4, 128, 700
    kc = torch.randn(B, S + 1, hkv, d, device="cuda").bfloat16()
    vc = torch.randn(B, S + 1, hkv, d, device="cuda").bfloat16()
    kc0, vc0 = kc.clone(), vc.clone()
    q = torch.randn(B, hkv * G, d, device="cuda")
    kn = torch.randn(B, hkv, d, device="cuda").bfloat16()
    vn = torch.randn(B, hkv, d, device="cuda").bfloat16()
    sl = torch.full((B,), S, dtype=torch.int32, device="cuda")
    act = torch.tensor([1, 0, 1, 0], dtype=torch.int32, device="cuda")
    out = torch.full((B, hkv * G, d), 7.0, device="cuda")
    kernels.decode_attention_rows(q, kc, vc, sl, S + 1, act, k_new=kn, v_new=vn, out=out, advance=sl)
    ref = kernels.decode_attention(q, kc0.clone(), vc0.clone(), torch.full((B,), S, dtype=torch.int32, device="cuda"),
                                   S + 1, k_new=kn, v_new=vn)
    torch.cuda.synchronize()
    assert sl.tolist() == [S + 1, S, S + 1, S]
    for b in (1, 3):
        assert torch.equal(kc[b], kc0[b]) and torch.equal(vc[b], vc0[b])
        assert torch.all(out[b] == 7.0)
    for b in (0, 2):
        torch.testing.assert_close(out[b], ref[b], rtol=1e-5, atol=1e-6)
    # out projection + lm_head with the mask
    D = 512
    w = kernels.pack_weight((torch.randn(D, D, device="cuda") / D ** 0.5).bfloat16())
    a = torch.randn(B, D, device="cuda")
    x = torch.randn(B, D, device="cuda")
    x0 = x.clone()
    kernels.out_proj(a, w, x, row_active=act)
    torch.cuda.synchronize()
    assert torch.equal(x[1], x0[1]) and torch.equal(x[3], x0[3])
    assert not torch.equal(x[0], x0[0])
    V = 258
    emb = torch.randn(V, D, device="cuda").bfloat16()
    tok = torch.full((B,), 3, dtype=torch.int32, device="cuda")
    pos = torch.full((B,), 10, dtype=torch.int32, device="cuda")
    log = torch.zeros((B, 8), dtype=torch.int32, device="cuda")
    xn = x.clone()
    kernels.lm_head(x, kernels.pack_weight(emb.t().contiguous()), V, emb, xn, tok, pos, tokens_log=log, log_stride=8,
                    row_active=act, log_pos_base=8)
    torch.cuda.synchronize()
    assert pos.tolist() == [11, 10, 11, 10] and tok[1] == 3 and tok[3] == 3
    assert torch.equal(xn[1], x[1])
    assert log[0, 3] == tok[0] and log[2, 3] == tok[2] and int(log[1].abs().sum()) == 0
