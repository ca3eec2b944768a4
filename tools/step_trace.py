"""Per-phase timeline of the persistent decode step (needs a librk built with
-DSTP_TRACE: SRC=step tools/build_variant.sh strace -DSTP_TRACE).  Runs a few
C2 token steps and prints, per phase, the mean / max over CTAs of the time
each CTA spent (us), averaged over layers, from the last launch.

    ROUNDKV_B200_LIB=variants_tmp/librk_strace.so python tools/step_trace.py --batch 1
"""
import argparse
import ctypes as C
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from bench import WORKLOADS  # noqa: E402
from paper_2502_15294_b200 import _lib, kernels  # noqa: E402
from paper_2502_15294_b200.decode_engine import EngineConfig, RoundDecodeEngine  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="c2")
ap.add_argument("--batch", type=int, default=1)
a = ap.parse_args()
w = dict(WORKLOADS[a.workload])
w.update(batch=a.batch, decode_steps=8, plant=0, host_unique=1, step_kernel="persistent")
eng = RoundDecodeEngine(EngineConfig(**w))
eng.lower_len.copy_(eng.lower_len0)
eng.upper_len.copy_(eng.upper_len0)
eng.pos.copy_(eng.pos_dec0)
for t in range(6):
    kernels.decode_step(eng.step_args[t])
torch.cuda.synchronize()
G = torch.cuda.get_device_properties(0).multi_processor_count
L = eng.cfg.num_layers
n = 160 * 64 * 10
buf = (C.c_ulonglong * n)()
_lib.lib.rk_debug_step_trace.argtypes = [C.c_void_p, C.c_int]
assert _lib.lib.rk_debug_step_trace(buf, n) == 0
tr = np.frombuffer(buf, dtype=np.uint64).reshape(160, 64, 10)[:G, :L].astype(np.int64)
t0 = tr[:, 0, 0].min()
tr = (tr - t0) / 1000.0        # us
names = {"qkv_stage": (0, 1), "qkv_tiles": (1, 2), "wait_qkv": (2, 3), "att": (3, 4), "mrg+wait": (4, 5),
         "wait_mrg": (5, 6), "out_stage": (6, 7), "out_tiles": (7, 8), "wait_out(next)": (8, None)}
res = {"batch": a.batch, "step_us": round(float(tr[:, L - 1, 8].max()), 1)}
for k, (i, j) in names.items():
    if j is None:
        d = tr[:, 1:, 0] - tr[:, :-1, 8]
    else:
        d = tr[:, :, j] - tr[:, :, i]
    res[k] = [round(float(d.mean()), 2), round(float(d.max(axis=0).mean()), 2)]
# producer: when it finished issuing layer l vs when consumers finished it
res["prod_ahead_us"] = round(float((tr[:, :, 8] - tr[:, :, 9]).mean()), 2)
res["layer_us"] = round(float(np.diff(tr[:, :, 8].max(axis=0)).mean()), 2)
print(json.dumps(res))
