"""The drop-in engine's own invariants, mirroring the reference's engine tests
(SURVEY §8c: test_engine.py:108-119 incremental == batch, :206-229 masked ==
spliced): a teacher-forced prefill equals the same tokens fed one at a time, and
attention over a spliced cache equals attention over the full cache with the
dropped positions masked (engine.py:94-112 — the basis of round splicing)."""

from __future__ import annotations

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2502_15294_b200.engine import Model, ModelConfig  # noqa: E402


def _model():
    return Model(ModelConfig(num_layers=3, num_heads=4, d_model=64, rng_seed=3))


def test_incremental_equals_batch_prefill():
    model = _model()
    L = model.config.num_layers
    toks = [int(x) for x in np.random.default_rng(1).integers(0, 256, size=24)]
    batch_cache = model.new_cache()
    hb, _ = model.forward_range(batch_cache, 0, L, tokens=toks, positions=np.arange(len(toks)))
    inc_cache = model.new_cache()
    rows = []
    for i, t in enumerate(toks):
        h, _ = model.forward_range(inc_cache, 0, L, tokens=[t], positions=[i])
        rows.append(h)
    hi = torch.cat(rows)
    torch.testing.assert_close(hi, hb, rtol=1e-4, atol=1e-4)
    for l in range(L):
        torch.testing.assert_close(inc_cache.layer(l).keys, batch_cache.layer(l).keys, rtol=1e-4, atol=1e-4)
        assert torch.equal(inc_cache.layer(l).positions, batch_cache.layer(l).positions)


def test_spliced_cache_equals_masked_attention():
    model = _model()
    L = model.config.num_layers
    rng = np.random.default_rng(2)
    toks = [int(x) for x in rng.integers(0, 256, size=40)]
    cache = model.new_cache()
    model.forward_range(cache, 0, L, tokens=toks, positions=np.arange(len(toks)))
    keep = np.concatenate([np.arange(0, 10), np.arange(22, 40)])           # drop positions 10..21
    spliced = cache.spliced(keep)
    q_tok, q_pos = [7, 99, 3], [40, 41, 42]
    h_s, _ = model.forward_range(spliced, 0, L, tokens=q_tok, positions=q_pos)
    keep_set = torch.zeros(64, dtype=torch.bool, device=model.device)
    keep_set[torch.as_tensor(keep, device=model.device)] = True
    keep_set[40:] = True                                                    # the new rows stay visible

    def allowed(l, positions):
        return keep_set[positions]

    h_m, _ = model.forward_range(cache, 0, L, tokens=q_tok, positions=q_pos, allowed_fn=allowed)
    torch.testing.assert_close(h_s, h_m, rtol=1e-5, atol=1e-5)
