"""Time the C3 turn's phases on one engine (device events + host wall): the question's
lower layers (prefill + fused scoring), the selection round trip, the gather, the
question's upper layers, the answer loop.

    python tools/c3_phases.py [--batch 8] [--turns 3]
"""
import argparse
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from bench import WORKLOADS  # noqa: E402
from paper_2502_15294_b200.decode_engine import EngineConfig, RoundDecodeEngine  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--batch", type=int, default=8)
ap.add_argument("--turns", type=int, default=3)
ap.add_argument("--workload", default="c3")
a = ap.parse_args()
w = dict(WORKLOADS[a.workload])
w["batch"] = a.batch
eng = RoundDecodeEngine(EngineConfig(**w))
eng.prepare()
torch.cuda.synchronize()
for t in range(a.turns):
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(6)]
    h = []
    with torch.cuda.stream(eng.compute_stream):
        h.append(time.perf_counter())
        ev[0].record()
        eng._set_question()
        eng.graph_a.replay()
        ev[1].record()
        kept = eng._select_to_host()
        h.append(time.perf_counter())
        ev[2].record()
        eng.copy_stream.wait_stream(eng.compute_stream)
        eng.issue_gather(eng.gather_plan(kept))
        ev[3].record()
        eng._phase_b1(layer_wait=True)
        ev[4].record()
        h.append(time.perf_counter())
        eng.graph_b.replay()
        ev[5].record()
        torch.cuda.synchronize()
        h.append(time.perf_counter())
    names = ["phaseA", "select_sync", "gather_issue", "upper_question", "answer_loop"]
    print(t, {n: round(ev[i].elapsed_time(ev[i + 1]), 2) for i, n in enumerate(names)},
          "host_ms", [round(1000 * (h[i + 1] - h[i]), 1) for i in range(len(h) - 1)],
          "refined", eng.refined_dialogues, "copied", eng.last_copied_rounds)
