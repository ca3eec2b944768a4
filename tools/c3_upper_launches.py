"""One C3 turn's upper-question phase inside an NVTX range "upper" (for an ncu launch list):
    ncu --nvtx --nvtx-include "upper/" --metrics gpu__time_duration.sum --csv python tools/c3_upper_launches.py"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from bench import WORKLOADS  # noqa: E402
from paper_2502_15294_b200.decode_engine import EngineConfig, RoundDecodeEngine  # noqa: E402

eng = RoundDecodeEngine(EngineConfig(**dict(WORKLOADS["c3"])))
eng.prepare()
torch.cuda.synchronize()
with torch.cuda.stream(eng.compute_stream):
    eng._set_question()
    eng.graph_a.replay()
    kept = eng._select_to_host()
    eng.copy_stream.wait_stream(eng.compute_stream)
    eng.issue_gather(eng.gather_plan(kept))
    torch.cuda.synchronize()          # gathers done: the range times the upper layers alone
    torch.cuda.nvtx.range_push("upper")
    eng._phase_b1(layer_wait=True)
    torch.cuda.synchronize()
    torch.cuda.nvtx.range_pop()
print("ok")
