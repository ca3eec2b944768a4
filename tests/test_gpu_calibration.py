"""GPU watershed calibration (calibration.py) against the
reference's own calibration outputs (tests/golden/calib_cases.npz, generated
by tools/make_golden.py from pipeline.capture_all_layers + layer_distributions
+ stats.kl_curve + detect_watershed, pipeline.py:439-494): the per-layer round
distributions come from one device prefill with fused scoring (no capture
matrices) and must match the reference's, and the detected layers must be
identical."""

from __future__ import annotations

import numpy as np
import pytest

from conftest import GOLDEN

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2502_15294_b200 import calibration as cal  # noqa: E402
from paper_2502_15294_b200.engine import Model, ModelConfig  # noqa: E402
from paper_2502_15294_b200.stats import Round  # noqa: E402


def _corpus(z):
    convs = []
    for i in range(int(z["n_conv"])):
        spans = z[f"c{i}_spans"]
        rounds = [Round(m, (int(s[0][0]), int(s[0][1])), (int(s[1][0]), int(s[1][1]))) for m, s in enumerate(spans)]
        convs.append(cal.Conversation(rounds=rounds, token_ids=[int(t) for t in z[f"c{i}_ids"]]))
    return convs


def test_calibration_matches_reference():
    z = np.load(GOLDEN / "calib_cases.npz")
    model = Model(ModelConfig(num_layers=int(z["num_layers"]), num_heads=int(z["num_heads"]),
                              d_model=int(z["d_model"]), rng_seed=int(z["seed"])))
    convs = _corpus(z)
    curves = []
    for i, conv in enumerate(convs):
        n = cal.analysis_round_index(conv)
        assert n == int(z[f"c{i}_n"])
        masses = cal.layer_round_masses(model, conv, n)
        np.testing.assert_allclose(masses, z[f"c{i}_masses"], rtol=1e-4, atol=1e-7)
        curve = cal.kl_curve(masses)
        np.testing.assert_allclose(curve.values, z[f"c{i}_curve"], rtol=1e-3, atol=1e-7)
        curves.append(curve)
    assert cal.detect_watershed(curves).layer == int(z["ws_max_drop_0.1"])
    res = cal.calibrate_watershed(model, convs, criterion="threshold", tau=1e-3)
    assert res.layer == int(z["ws_threshold_0.001"]) and res.corpus_size == len(convs)


def test_calibration_pre_capture_matches_reference():
    """capture_mode="pre" (softmax of the head-summed logits, engine.py:187-200):
    the per-layer round distributions of every conversation equal the
    reference's capture_all_layers + layer_distributions."""
    z = np.load(GOLDEN / "calib_cases.npz")
    model = Model(ModelConfig(num_layers=int(z["num_layers"]), num_heads=int(z["num_heads"]),
                              d_model=int(z["d_model"]), rng_seed=int(z["seed"]), capture_mode="pre"))
    for i, conv in enumerate(_corpus(z)):
        n = cal.analysis_round_index(conv)
        masses = cal.layer_round_masses(model, conv, n)
        np.testing.assert_allclose(masses, z[f"c{i}_masses_pre"], rtol=1e-4, atol=1e-7)


@pytest.mark.parametrize("mode", ["post", "pre"])
def test_reference_calibration_entry_points(mode):
    """The reference module names (pipeline.capture_all_layers, layer_distributions,
    conversation_kl_curve; stats.kl_curve): the materialised route gives the
    golden distributions and curves too."""
    from paper_2502_15294_b200 import pipeline as pl
    from paper_2502_15294_b200 import stats as st
    z = np.load(GOLDEN / "calib_cases.npz")
    model = Model(ModelConfig(num_layers=int(z["num_layers"]), num_heads=int(z["num_heads"]),
                              d_model=int(z["d_model"]), rng_seed=int(z["seed"]), capture_mode=mode))
    key = "masses" if mode == "post" else "masses_pre"
    for i, conv in enumerate(_corpus(z)):
        n = pl.analysis_round_index(conv)
        caps = pl.capture_all_layers(model, conv)
        dists = pl.layer_distributions([caps[l] for l in range(int(z["num_layers"]))], conv.rounds, n)
        masses = np.stack([np.asarray(d.masses) for d in dists])
        np.testing.assert_allclose(masses, z[f"c{i}_{key}"], rtol=1e-4, atol=1e-7)
        if mode == "post":
            np.testing.assert_allclose(st.kl_curve(masses).values, z[f"c{i}_curve"], rtol=1e-3, atol=1e-7)
            np.testing.assert_allclose(pl.conversation_kl_curve(model, conv).values, z[f"c{i}_curve"],
                                       rtol=1e-3, atol=1e-7)
