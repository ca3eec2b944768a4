"""Run a few engine turns (for ncu launch lists / captures).

    python tools/profile_engine.py --workload c2 --decode-steps 4 --turns 2
"""
import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from bench import WORKLOADS  # noqa: E402
from paper_2502_15294_b200.decode_engine import EngineConfig, RoundDecodeEngine  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="c2")
ap.add_argument("--decode-steps", type=int, default=4)
ap.add_argument("--turns", type=int, default=2)
ap.add_argument("--batch", type=int, default=None)
ap.add_argument("--eager", action="store_true")
ap.add_argument("--profile-turns", action="store_true",
                help="cudaProfilerStart/Stop around the turns (ncu --profile-from-start off)")
a = ap.parse_args()
w = dict(WORKLOADS[a.workload])
w["decode_steps"] = a.decode_steps
if a.batch:
    w["batch"] = a.batch
eng = RoundDecodeEngine(EngineConfig(**w))
if not a.eager:
    eng.prepare(e2e=False)
torch.cuda.synchronize()
if a.profile_turns:
    torch.cuda.profiler.start()
if a.eager:
    with torch.cuda.stream(eng.compute_stream):
        for _ in range(a.turns):
            eng.run_turn_eager()
else:
    for _ in range(a.turns):
        eng.run_turn()
torch.cuda.synchronize()
if a.profile_turns:
    torch.cuda.profiler.stop()
print("turns done", eng.turn_breakdown_ms() if not a.eager else "")
