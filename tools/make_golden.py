"""Generate golden vectors for the round-attention hot path from the REAL
reference package (`/root/reference/pkg`), imported in the build container.

The reference is copied to a scratch dir, its Cython kernel built in place
(`setup.py build_ext --inplace`, exactly as SURVEY.md §8c describes), and the
package imported under the alias `roundkv_ref`.  Outputs go to
`tests/golden/` as small .npz / .json fixtures that travel with the repo;
`/root/reference` is never read at test time.

    python tools/make_golden.py            # regenerate all fixtures
"""

from __future__ import annotations

import importlib.util
import json
import os
import shutil
import subprocess
import sys
import tempfile
from pathlib import Path

import numpy as np

REPO = Path(__file__).resolve().parents[1]
GOLDEN = REPO / "tests" / "golden"
REF_PKG = Path("/root/reference/pkg")


def load_reference():
    scratch = Path(tempfile.mkdtemp(prefix="rk_ref_"))
    dst = scratch / "pkg"
    shutil.copytree(REF_PKG, dst)
    subprocess.run([sys.executable, "setup.py", "build_ext", "--inplace"], cwd=dst,
                   check=True, capture_output=True)
    src = dst / "src" / "roundkv"
    spec = importlib.util.spec_from_file_location(
        "roundkv_ref", src / "__init__.py", submodule_search_locations=[str(src)])
    mod = importlib.util.module_from_spec(spec)
    sys.modules["roundkv_ref"] = mod
    spec.loader.exec_module(mod)
    import roundkv_ref.backend as backend  # noqa: E402
    assert backend.BACKEND_NAME == "ext", backend.BACKEND_NAME
    return mod


def bf16(x):
    sys.path.insert(0, str(REPO))
    from oracle.attention import round_to_bf16
    return round_to_bf16(x)


def kernel_cases(ref, rng):
    """attention_forward contract cases (MHA; GQA by expansion is a test-side
    transform).  Mix of the reference test shapes (test_backend.py:8-21) and
    larger bf16-rounded cases."""
    from roundkv_ref.backend import attention_forward
    cases = {}
    specs = []
    for t in range(24):
        n = int(rng.integers(1, 9))
        s = int(rng.integers(n, 80))
        h = int(rng.choice([1, 2, 4, 8]))
        d = int(rng.choice([2, 8, 16, 64]))
        specs.append((n, s, h, d, t % 2 == 1, t % 3 == 0, False))
    specs += [(1, 1, 1, 2, False, True, False), (5, 12, 4, 8, True, True, False),
              (1, 512, 8, 64, False, True, True), (32, 300, 8, 64, False, True, True),
              (1, 600, 4, 128, True, True, True), (16, 300, 2, 128, False, True, True),
              (3, 40, 8, 64, True, False, True)]
    for idx, (n, s, h, d, masked, capture, use_bf16) in enumerate(specs):
        q = rng.standard_normal((n, h, d)).astype(np.float32)
        k = rng.standard_normal((s, h, d)).astype(np.float32)
        v = rng.standard_normal((s, h, d)).astype(np.float32)
        if use_bf16:
            q, k, v = bf16(q), bf16(k), bf16(v)
        q_pos = np.arange(s - n, s, dtype=np.int64)
        k_pos = np.arange(s, dtype=np.int64)
        allowed = None
        if masked:
            allowed = rng.random(s) < 0.6
            allowed[s - n:] = True
        out, scores = attention_forward(q, k, v, q_pos, k_pos, allowed=allowed, capture=capture)
        p = f"c{idx}_"
        if use_bf16:   # exactly bf16-representable: store the upper halves only
            for name, arr in (("q", q), ("k", k), ("v", v)):
                cases[p + name + "_bf16"] = (arr.view(np.uint32) >> 16).astype(np.uint16)
        else:
            cases[p + "q"], cases[p + "k"], cases[p + "v"] = q, k, v
        cases[p + "q_pos"], cases[p + "k_pos"] = q_pos, k_pos
        cases[p + "allowed"] = allowed if allowed is not None else np.ones(0, bool)
        cases[p + "masked"] = np.array(masked)
        cases[p + "capture"] = np.array(capture)
        cases[p + "out"] = out
        cases[p + "scores"] = scores if scores is not None else np.zeros((0, 0))
    cases["count"] = np.array(len(specs))
    np.savez_compressed(GOLDEN / "kernel_cases.npz", **cases)


def stats_cases(ref, rng):
    from roundkv_ref.conversation import Round
    from roundkv_ref.stats import aggregate_round_attention, normalize
    out = {}
    count = 0
    for t in range(40):
        layout = [(int(rng.integers(1, 6)), int(rng.integers(1, 6))) for _ in range(int(rng.integers(2, 7)))]
        if t % 4 == 0:
            layout[-1] = (layout[-1][0], 0)      # in-flight question (pipeline shape)
        rounds, pos = [], 0
        for m, (ql, al) in enumerate(layout):
            rounds.append(Round(m, (pos, pos + ql), (pos + ql, pos + ql + al)))
            pos += ql + al
        n = len(rounds) - 1
        seq = rounds[-1].q_span[1] if t % 4 == 0 else rounds[-1].end
        mat = np.zeros((seq, seq))
        for i in range(seq):
            row = rng.random(i + 1)
            if t % 7 == 3 and i >= 2:
                row[: i // 2] = 0.0
            mat[i, : i + 1] = row / row.sum()
        row_offset = rounds[-1].q_span[0] if t % 2 == 0 else 0
        scores = mat[row_offset:]
        active = list(range(n))
        if t % 5 == 4 and n > 1:
            active = [a for a in active if a != int(rng.integers(0, n))]
        raw = aggregate_round_attention(scores, rounds, "question", n,
                                        active_rounds=active, row_offset=row_offset)
        dist = normalize(raw, layer=1, round_indices=active)
        p = f"s{count}_"
        out[p + "layout"] = np.array(layout, dtype=np.int64)
        out[p + "scores"] = scores
        out[p + "row_offset"] = np.array(row_offset)
        out[p + "active"] = np.array(active, dtype=np.int64)
        out[p + "raw"] = raw
        out[p + "masses"] = dist.masses
        out[p + "degenerate"] = np.array(dist.degenerate)
        count += 1
    out["count"] = np.array(count)
    np.savez_compressed(GOLDEN / "stats_cases.npz", **out)


def select_cases(ref, rng):
    from roundkv_ref.selection import SelectionPolicy, select
    from roundkv_ref.stats import normalize
    raws = []
    for t in range(120):
        n = int(rng.integers(1, 200))
        kind = t % 6
        if kind == 0:
            raw = rng.random(n)
        elif kind == 1:
            raw = rng.integers(0, 4, size=n).astype(np.float64)        # heavy ties
        elif kind == 2:
            raw = np.zeros(n)                                          # degenerate
        elif kind == 3:
            base = rng.random(max(1, n // 3))
            raw = np.resize(base, n)                                   # duplicated values
        elif kind == 4:
            raw = rng.random(n) ** 8 * 1e-3                            # skewed small
        else:
            raw = np.full(n, 0.1)                                      # all equal
        raws.append(raw)
    raws += [np.array([.5, .05, .3, .15]), np.full(20, 1 / 20), np.array([.7, .1, .1, .1]),
             np.array([.3, .2, .3, .2]), np.array([1e-300, 2e-300, 0.0]),
             np.array([0.1] * 30), np.array([0.1] * 10)]
    policies = [("top_percent", dict(fraction=0.10)), ("top_percent", dict(fraction=0.30)),
                ("top_percent", dict(fraction=0.5, min_rounds=3)), ("top_percent", dict(fraction=1.0)),
                ("top_percent", dict(fraction=0.05)), ("fixed", dict(v=0.1)), ("fixed", dict(v=0.01)),
                ("adaptive", dict(kappa=1.0)), ("adaptive", dict(kappa=0.0)),
                ("adaptive", dict(kappa=2.5)), ("all", {})]
    cases = []
    for raw in raws:
        dist = normalize(raw)
        results = []
        for kind, kw in policies:
            res = select(dist, SelectionPolicy(kind=kind, **kw))
            results.append(dict(kind=kind, params=kw, kept=list(res.kept)))
        cases.append(dict(raw=[float(x).hex() for x in raw],
                          masses=[float(x).hex() for x in dist.masses],
                          degenerate=bool(dist.degenerate), results=results))
    (GOLDEN / "select_cases.json").write_text(json.dumps(cases))


def store_memory_cases(ref, rng):
    from roundkv_ref.store import TieredStore, footprint_report, memory_ratio, save_percent
    from roundkv_ref.errors import RoundKVError
    memory = []
    for (L, lw, K, T) in [(24, 11, 2, 10), (4, 2, 1, 8), (32, 5, 4, 32), (28, 10, 7, 64),
                          (32, 5, 13, 128), (80, 18, 0, 5), (16, 5, 3, 3)]:
        memory.append(dict(args=[L, lw, K, T], ratio=memory_ratio(L, lw, K, T).hex(),
                           save=save_percent(L, lw),
                           fp={k: (float(v).hex() if isinstance(v, float) else v)
                               for k, v in footprint_report(1, 1024, 4096, L, lw, K, T).items()}))
    for row in json.loads((REF_PKG / "src/roundkv/data/model_watershed.json").read_text())["rows"]:
        memory.append(dict(table5=[row["layers"], row["watershed"]], save=save_percent(row["layers"], row["watershed"]),
                           published=row["save_percent"]))
    # random op sequences over the tiered store: ledger + tiers after each op
    sequences = []
    for t in range(30):
        L = int(rng.integers(3, 10))
        lw = int(rng.integers(1, L))
        d = int(rng.choice([8, 16, 32]))
        cap = int(rng.choice([1 << 14, 1 << 16, 1 << 20, 64 << 20]))
        evict = bool(t % 3 == 0)
        store = TieredStore(L, lw, d, device_capacity=cap, evict_lower_on_pressure=evict)
        ops, results = [], []
        stored = 0
        for step in range(int(rng.integers(5, 25))):
            r = rng.random()
            if r < 0.35 or stored == 0:
                tok = int(rng.integers(1, 40))
                op = ["put", stored, tok, bool(rng.random() < 0.5)]
                try:
                    store.put_round(stored, np.zeros((lw, 2, tok, d), np.float32),
                                    np.zeros((L - lw, 2, tok, d), np.float32), np.arange(tok),
                                    upper_on_device=op[3])
                    err = None
                    stored += 1
                except RoundKVError as e:
                    err = type(e).__name__
            elif r < 0.5:
                op = ["begin", step]
                store.begin_turn(step)
                err = None
            elif r < 0.65:
                sel = sorted(set(int(x) for x in rng.integers(0, stored + 1, size=int(rng.integers(1, 4)))))
                op = ["fetch_upper", sel]
                try:
                    store.fetch_upper(sel)
                    err = None
                except RoundKVError as e:
                    err = type(e).__name__
            elif r < 0.75:
                op = ["fetch_lower_all", stored]
                try:
                    store.fetch_lower_all(stored)
                    err = None
                except RoundKVError as e:
                    err = type(e).__name__
            elif r < 0.87:
                sel = sorted(set(int(x) for x in rng.integers(0, stored, size=int(rng.integers(1, 4)))))
                op = ["writeback_upper", sel]
                try:
                    store.writeback_upper(sel)
                    err = None
                except RoundKVError as e:
                    err = type(e).__name__
            elif r < 0.95:
                m = int(rng.integers(0, stored))
                op = ["drop_upper", m]
                store.drop_upper(m)
                err = None
            else:
                op = ["end_session"]
                store.end_session()
                err = None
            ops.append(op)
            results.append(dict(err=err, used=store.device_used_bytes,
                                ledger=[store.ledger.h2d_events, store.ledger.h2d_bytes,
                                        store.ledger.d2h_events, store.ledger.d2h_bytes],
                                per_turn=store.ledger.report_rows(),
                                tiers={f"{k[0]}:{k[1]}": b.tier for k, b in store.blocks.items()}))
        sequences.append(dict(L=L, lw=lw, d=d, cap=cap, evict=evict, ops=ops, results=results))
    (GOLDEN / "store_cases.json").write_text(json.dumps(dict(memory=memory, sequences=sequences)))


def pipeline_c1(ref, rng_unused, turns=9, steps=63):
    """C1 tiny config: Model(4 layers, 8 heads, d_model 512,
    seed 42), watershed 2, top_percent 0.10, 63 random byte ids per question
    from default_rng(0), max_decode_steps=63."""
    from roundkv_ref.engine import Model, ModelConfig
    from roundkv_ref.pipeline import RoundPipeline
    from roundkv_ref.selection import SelectionPolicy
    model = Model(ModelConfig(num_layers=4, num_heads=8, d_model=512, rng_seed=42))
    pipe = RoundPipeline(model, 2, policy=SelectionPolicy("top_percent", fraction=0.10))
    qrng = np.random.default_rng(0)
    out = {}
    questions = []
    for t in range(turns):
        q = [int(x) for x in qrng.integers(0, 256, size=63)]
        questions.append(q)
        res = pipe.run_turn(q, max_decode_steps=steps)
        m = res.metrics
        out[f"t{t}_answer"] = np.array(res.answer_ids, dtype=np.int64)
        out[f"t{t}_kept"] = np.array(m.kept, dtype=np.int64)
        if m.distribution is not None:
            out[f"t{t}_raw"] = m.distribution.raw
            out[f"t{t}_masses"] = m.distribution.masses
        out[f"t{t}_ledger"] = np.array([m.upper_h2d_events, m.upper_h2d_bytes, m.lower_h2d_events,
                                        m.lower_h2d_bytes, m.d2h_events, m.d2h_bytes,
                                        m.device_used_peak, m.hist_tokens, m.hist_tokens_attended,
                                        m.selection_invocations], dtype=np.int64)
    out["questions"] = np.array(questions, dtype=np.int64)
    out["turns"] = np.array(turns)
    out["steps"] = np.array(steps)
    # upper-layer KV of the last round, as a whole-state checksum
    last = pipe.store.get_block(turns - 1, "upper").payload
    out["last_upper_payload_sum"] = np.array([float(np.sum(last, dtype=np.float64))])
    np.savez_compressed(GOLDEN / "c1_pipeline.npz", **out)


def calibration_cases(ref, rng, n_conv=4):
    """Watershed calibration (pipeline.py:439-494, stats.py:118-181) on a
    6-layer model over synthetic conversations: per-conversation layer
    distributions and KL curves, and the corpus watershed for both criteria."""
    sys.path.insert(0, str(REPO))
    from oracle.rounds import make_conversation_layout
    from roundkv_ref.conversation import Conversation, Round, Token
    from roundkv_ref.engine import Model, ModelConfig
    from roundkv_ref.pipeline import analysis_round_index, capture_all_layers, layer_distributions
    from roundkv_ref.stats import detect_watershed, kl_curve
    model = Model(ModelConfig(num_layers=6, num_heads=4, d_model=128, rng_seed=7))
    model_pre = Model(ModelConfig(num_layers=6, num_heads=4, d_model=128, rng_seed=7, capture_mode="pre"))
    out = {"n_conv": np.array(n_conv), "num_layers": np.array(6), "num_heads": np.array(4),
           "d_model": np.array(128), "seed": np.array(7)}
    curves = []
    for i in range(n_conv):
        n_rounds = int(rng.integers(3, 7))
        q_lens = [int(x) for x in rng.integers(8, 40, size=n_rounds)]
        a_lens = [int(x) for x in rng.integers(10, 60, size=n_rounds)]
        if i % 2:                                  # odd conversations end with an in-flight question
            a_lens[-1] = 0
        ids, spans = make_conversation_layout(q_lens, a_lens, rng)
        conv = Conversation(rounds=[Round(m, tuple(q), tuple(a)) for m, (q, a) in enumerate(spans)],
                            tokens=[Token(t, p) for p, t in enumerate(ids)])
        n = analysis_round_index(conv)
        caps = capture_all_layers(model, conv)
        dists = layer_distributions([caps[l] for l in range(6)], conv.rounds, n)
        curve = kl_curve([d.masses for d in dists])
        curves.append(curve)
        out[f"c{i}_ids"] = np.array(ids, dtype=np.int64)
        out[f"c{i}_spans"] = np.array(spans, dtype=np.int64)
        out[f"c{i}_n"] = np.array(n)
        out[f"c{i}_masses"] = np.stack([d.masses for d in dists])
        caps_pre = capture_all_layers(model_pre, conv)          # head-summed-logit capture (engine.py:187-200)
        out[f"c{i}_masses_pre"] = np.stack([d.masses for d in layer_distributions([caps_pre[l] for l in range(6)],
                                                                                  conv.rounds, n)])
        out[f"c{i}_curve"] = curve.values
    for crit, tau in (("max_drop", 0.1), ("threshold", 0.1), ("threshold", 1e-3)):
        w = detect_watershed(curves, criterion=crit, tau=tau)
        out[f"ws_{crit}_{tau}"] = np.array(w.layer)
        out["mean_curve"] = w.curve.values
    np.savez_compressed(GOLDEN / "calib_cases.npz", **out)


def pipeline_variants(ref):
    """C1-shaped pipeline runs with the inactivity drop policy active
    (drop_window=2, selection.py:168-204 + store.drop_upper) and with the
    fixed / adaptive strategies (selection.py:76-108): 6 turns, 15 decode steps."""
    from roundkv_ref.engine import Model, ModelConfig
    from roundkv_ref.pipeline import RoundPipeline
    from roundkv_ref.selection import SelectionPolicy
    variants = {
        "drop2": dict(policy=SelectionPolicy("top_percent", fraction=0.25), drop_window=2, drop_protect=1),
        "fixed": dict(policy=SelectionPolicy("fixed", v=0.12)),
        "adaptive": dict(policy=SelectionPolicy("adaptive", kappa=0.5)),
        # the head-summed-logit capture (ModelConfig.capture_mode="pre", engine.py:187-200)
        "pre": dict(policy=SelectionPolicy("top_percent", fraction=0.25)),
        # full-cache baseline mode (pipeline.py:115-150, mode="baseline")
        "baseline": dict(mode="baseline"),
        # masked attention over every upper block instead of splicing (attend_mode="mask")
        "mask": dict(policy=SelectionPolicy("top_percent", fraction=0.25)),
    }
    out = {}
    for name, kw in variants.items():
        mode = "pre" if name == "pre" else "post"
        model = Model(ModelConfig(num_layers=4, num_heads=8, d_model=512, rng_seed=42, capture_mode=mode))
        pipe = RoundPipeline(model, 2, **kw)
        if name == "mask":
            pipe.attend_mode = "mask"
        qrng = np.random.default_rng(5)
        for t in range(6):
            q = [int(x) for x in qrng.integers(0, 256, size=31)]
            res = pipe.run_turn(q, max_decode_steps=15)
            m = res.metrics
            out[f"{name}_t{t}_q"] = np.array(q, dtype=np.int64)
            out[f"{name}_t{t}_answer"] = np.array(res.answer_ids, dtype=np.int64)
            out[f"{name}_t{t}_kept"] = np.array(m.kept, dtype=np.int64)
            out[f"{name}_t{t}_dropped"] = np.array(sorted(pipe.activity.dropped), dtype=np.int64)
            out[f"{name}_t{t}_ledger"] = np.array([m.upper_h2d_events, m.upper_h2d_bytes, m.d2h_events, m.d2h_bytes,
                                                   m.device_used_peak, m.hist_tokens_attended], dtype=np.int64)
    np.savez_compressed(GOLDEN / "c1_variants.npz", **out)


def main():
    GOLDEN.mkdir(parents=True, exist_ok=True)
    ref = load_reference()
    rng = np.random.default_rng(20250215)
    kernel_cases(ref, rng)
    stats_cases(ref, rng)
    select_cases(ref, rng)
    store_memory_cases(ref, rng)
    pipeline_c1(ref, rng)
    calibration_cases(ref, np.random.default_rng(777))
    pipeline_variants(ref)
    for p in sorted(GOLDEN.iterdir()):
        print(f"{p.name:28s} {p.stat().st_size:>10d} B")


if __name__ == "__main__":
    main()
