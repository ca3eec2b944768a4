"""C1 (BASELINE configs[0], the reference's own CPU-runnable case): whole turns
of the tiny model (4 layers, 8 heads, d_model 512, watershed 2, top_percent 0.10,
63-byte questions, 63 decode steps) through the GPU drop-in
RoundPipeline, timed per turn, beside the oracle port of the reference pipeline
(oracle/model.py, NumPy + the reference's compiled kernel where built) on this
box's CPU.  Both replay the golden conversation (tests/golden/c1_pipeline.npz)
and must produce its answers.

    python tools/bench_c1.py [--json out.json]
"""
import argparse
import json
import sys
import time
from pathlib import Path

REPO = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(REPO))
import numpy as np  # noqa: E402
import torch  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--json")
ap.add_argument("--cpu-turns", type=int, default=9)
a = ap.parse_args()
z = np.load(REPO / "tests" / "golden" / "c1_pipeline.npz")
turns, steps = int(z["turns"]), int(z["steps"])

from paper_2502_15294_b200.engine import Model, ModelConfig  # noqa: E402
from paper_2502_15294_b200.pipeline import RoundPipeline  # noqa: E402
from paper_2502_15294_b200.selection import SelectionPolicy  # noqa: E402


def gpu_run():
    model = Model(ModelConfig(num_layers=4, num_heads=8, d_model=512, rng_seed=42))
    pipe = RoundPipeline(model, 2, policy=SelectionPolicy("top_percent", fraction=0.10))
    ms, ok = [], True
    for t in range(turns):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        res = pipe.run_turn(list(z["questions"][t]), max_decode_steps=steps)
        torch.cuda.synchronize()
        ms.append(1000 * (time.perf_counter() - t0))
        ok &= list(res.answer_ids) == list(z[f"t{t}_answer"])
    return ms, ok


gpu_run()                                   # warm-up (kernel attributes, allocator)
g_ms, g_ok = gpu_run()

from oracle import model as om  # noqa: E402
from oracle import rounds as orr  # noqa: E402

model = om.Model(om.ModelConfig(num_layers=4, num_heads=8, d_model=512, rng_seed=42))
pipe = om.Pipeline(model, 2, orr.SelectionPolicy("top_percent", fraction=0.10))
c_ms, c_ok = [], True
for t in range(a.cpu_turns):
    t0 = time.perf_counter()
    res = pipe.run_turn(list(z["questions"][t]), max_decode_steps=steps)
    c_ms.append(1000 * (time.perf_counter() - t0))
    c_ok &= list(res["answer_ids"]) == list(z[f"t{t}_answer"])
out = dict(config="c1: L=4 H=8 d_model=512 Lw=2 top_percent 0.10, 9 turns x (63-byte question + 63 decode steps)",
           gpu_ms_per_turn=g_ms, gpu_answers_match=bool(g_ok), gpu_tokens_per_s=turns * (steps + 1) / (sum(g_ms) / 1e3),
           cpu_oracle_ms_per_turn=c_ms, cpu_answers_match=bool(c_ok),
           cpu_tokens_per_s=len(c_ms) * (steps + 1) / (sum(c_ms) / 1e3), cpu_threads=1,
           speedup_last_turn=c_ms[-1] / g_ms[len(c_ms) - 1])
print(json.dumps(out))
if a.json:
    Path(a.json).write_text(json.dumps(out, indent=1))
