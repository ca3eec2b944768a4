"""Host-side KL / watershed logic of calibration.py (re-exported under the
reference's stats names), checked against the properties the reference's own
test_stats.py pins (TestKL, TestKLCurve, TestWatershed; stats.py:118-181).
CPU only: these are NumPy restatements, no device work."""

from __future__ import annotations

import math

import numpy as np
import pytest

from paper_2502_15294_b200 import stats
from paper_2502_15294_b200.errors import DomainError

KLCurve, kl_divergence, kl_curve = stats.KLCurve, stats.kl_divergence, stats.kl_curve
detect_watershed, mean_curve = stats.detect_watershed, stats.mean_curve


def test_kl_identity_ln2_nonnegative_and_mismatch(rng):
    p = rng.dirichlet(np.ones(6))
    assert kl_divergence(p, p.copy()) == 0.0
    assert abs(kl_divergence(np.array([1.0, 0.0]), np.array([0.5, 0.5])) - math.log(2)) <= 1e-6
    for _ in range(300):
        n = int(rng.integers(2, 12))
        a, b = rng.dirichlet(np.ones(n)), rng.dirichlet(np.ones(n))
        assert kl_divergence(a, b) >= 0.0
    a, b = rng.dirichlet(np.ones(5)), rng.dirichlet(np.ones(5))
    assert kl_divergence(a, b) > 0.0
    with pytest.raises(DomainError):
        kl_divergence(np.ones(2) / 2, np.ones(3) / 3)


def test_kl_curve_composition_and_errors(rng):
    d = np.array([0.25, 0.25, 0.5])
    np.testing.assert_array_equal(kl_curve([d, d.copy(), d.copy(), d.copy()]).values, np.zeros(3))
    p0, p1, p2 = (rng.dirichlet(np.ones(5)) for _ in range(3))
    a, b, c = kl_divergence(p0, p1), kl_divergence(p0, p2), kl_divergence(p1, p2)
    np.testing.assert_allclose(kl_curve([p0, p1, p2]).values, [(a + b) / 2, c])
    assert np.all(kl_curve([rng.dirichlet(np.ones(8)) for _ in range(6)]).values >= 0.0)
    with pytest.raises(DomainError):
        kl_curve([np.ones(3) / 3])
    with pytest.raises(DomainError):
        kl_curve([np.ones(3) / 3, np.ones(4) / 4])


def _curves(num_layers, stable_from, seeds):
    out = []
    for seed in seeds:
        r = np.random.default_rng(seed)
        stable = r.dirichlet(np.ones(40))
        out.append(kl_curve([r.dirichlet(np.ones(40)) if l < stable_from else stable for l in range(num_layers)]))
    return out


def test_watershed_detection_properties():
    res = detect_watershed(_curves(12, 5, range(8)))
    assert res.layer == 5 and res.corpus_size == 8
    assert detect_watershed([KLCurve(values=np.full(7, 0.3), num_layers=8)]).layer == 1
    with pytest.raises(DomainError):
        detect_watershed([])
    cs = _curves(16, 7, range(6))
    assert detect_watershed(cs).layer == detect_watershed(list(reversed(cs))).layer == 7
    steep = KLCurve(values=np.array([2.0, 1.5, 0.04, 0.03, 0.02]), num_layers=6)
    assert detect_watershed([steep], criterion="threshold", tau=0.1).layer == 2
    never = KLCurve(values=np.array([2.0, 1.5, 0.8, 0.5, 0.9]), num_layers=6)
    assert detect_watershed([never], criterion="threshold", tau=0.1).layer == 3
    assert 0 < detect_watershed(_curves(24, 9, range(4))).layer < 24
    with pytest.raises(DomainError):
        detect_watershed(_curves(8, 3, [0]), criterion="magic")
    c1 = KLCurve(values=np.array([1.0, 0.0]), num_layers=3)
    c2 = KLCurve(values=np.array([3.0, 2.0]), num_layers=3)
    np.testing.assert_array_equal(mean_curve([c1, c2]).values, [2.0, 1.0])
