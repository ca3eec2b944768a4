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
    def allowed(l, positions):                     # NumPy key positions, as in the reference
        return np.isin(positions, list(keep) + q_pos)

    h_m, _ = model.forward_range(cache, 0, L, tokens=q_tok, positions=q_pos, allowed_fn=allowed)
    torch.testing.assert_close(h_s, h_m, rtol=1e-5, atol=1e-5)


def _prefill(model, tokens, capture_layers=None):
    cache = model.new_cache()
    h, caps = model.forward_range(cache, 0, model.config.num_layers, tokens=list(tokens),
                                  positions=np.arange(len(tokens)), capture_layers=capture_layers)
    return cache, h, caps


def test_config_validation_and_seeding():
    from paper_2502_15294_b200.errors import DomainError
    a, b = _model(), _model()
    assert all(torch.equal(x, y) for x, y in zip(a.w_q, b.w_q))
    c = Model(ModelConfig(num_layers=3, num_heads=4, d_model=64, rng_seed=4))
    assert not torch.equal(a.w_q[0], c.w_q[0])
    for kw in (dict(d_model=30, num_heads=4), dict(d_model=12, num_heads=4), dict(num_layers=0)):
        with pytest.raises(DomainError):
            ModelConfig(**kw)


def test_layer_partitions_compose_and_empty_tokens():
    from paper_2502_15294_b200.errors import DomainError
    model = _model()
    L = model.config.num_layers
    toks = [int(x) for x in np.random.default_rng(3).integers(0, 256, size=10)]
    _, whole, _ = _prefill(model, toks)
    for split in range(1, L):
        cache = model.new_cache()
        pos = np.arange(len(toks))
        mid, _ = model.forward_range(cache, 0, split, tokens=toks, positions=pos)
        h, _ = model.forward_range(cache, split, L, hidden=mid, positions=pos)
        torch.testing.assert_close(h, whole, rtol=1e-5, atol=1e-5)
    cache = model.new_cache()
    h, caps = model.forward_range(cache, 0, L, tokens=[], positions=[], capture_layers=[0])
    assert tuple(h.shape) == (0, model.config.d_model) and caps == {} and cache.lengths() == [0] * L
    with pytest.raises(DomainError, match="range"):
        model.forward_range(model.new_cache(), 0, L + 1, tokens=[1], positions=[0])
    with pytest.raises(DomainError):
        model.forward_range(model.new_cache(), 0, L, positions=[0])


def test_deterministic_and_capture_rows_normalised():
    model = _model()
    L = model.config.num_layers
    toks = [int(x) for x in np.random.default_rng(4).integers(0, 256, size=12)]
    _, h1, c1 = _prefill(model, toks, capture_layers=[L - 1])
    _, h2, c2 = _prefill(model, toks, capture_layers=[L - 1])
    assert torch.equal(h1, h2)
    s1 = c1[L - 1]
    s1 = s1.cpu().numpy() if hasattr(s1, "cpu") else np.asarray(s1)
    s2 = c2[L - 1]
    s2 = s2.cpu().numpy() if hasattr(s2, "cpu") else np.asarray(s2)
    assert np.array_equal(s1, s2)
    np.testing.assert_allclose(s1.sum(axis=1), 1.0, atol=1e-12)
    assert np.all(np.triu(s1, k=1) == 0.0)                         # causal
    pre = Model(ModelConfig(num_layers=3, num_heads=4, d_model=64, rng_seed=3, capture_mode="pre"))
    _, _, cp = _prefill(pre, toks, capture_layers=[1])
    sp = cp[1].cpu().numpy() if hasattr(cp[1], "cpu") else np.asarray(cp[1])
    np.testing.assert_allclose(sp.sum(axis=1), 1.0, atol=1e-12)
    assert np.all(np.triu(sp, k=1) == 0.0)


def test_decode_step_contract():
    from paper_2502_15294_b200.errors import DomainError
    model = _model()
    toks = [int(x) for x in np.random.default_rng(5).integers(0, 256, size=6)]
    ca, _, _ = _prefill(model, toks)
    cb, _, _ = _prefill(model, toks)
    a, _ = model.decode_step(ca, 7, 6)
    b, _ = model.decode_step(cb, 7, 6)
    assert a == b
    before = ca.lengths()
    model.decode_step(ca, 3, 7)
    assert ca.lengths() == [n + 1 for n in before]
    with pytest.raises(DomainError, match="non-empty"):
        model.decode_step(model.new_cache(), 3, 0)
