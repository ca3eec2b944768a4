"""Per-CTA timeline of the last projection launch in a CUDA graph of 32
(needs a librk built with -DPJ_TRACE: SRC=proj tools/build_variant.sh trace -DPJ_TRACE).

    ROUNDKV_B200_LIB=variants_tmp/librk_trace.so python tools/proj_trace.py --batch 1 --which qkv
"""
import argparse
import ctypes as C
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2502_15294_b200 import _lib, kernels  # noqa: E402
from paper_2502_15294_b200.decode_model import DecodeModel, ModelShape  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--batch", type=int, default=1)
ap.add_argument("--which", default="qkv")
a = ap.parse_args()
sh = ModelShape()
m = DecodeModel(sh, "cuda", seed=1)
B, D = a.batch, sh.d_model
x = torch.randn((B, D), device="cuda")
q = torch.zeros((B, sh.hq, sh.head_dim), device="cuda")
kv = torch.zeros((2, B, sh.hkv * sh.head_dim), dtype=torch.bfloat16, device="cuda")
pos = torch.zeros(B, dtype=torch.int32, device="cuda")
ws = kernels.proj_workspace(B, D, sh.qkv_width, "cuda")


def run():
    for l in range(sh.num_layers):
        if a.which == "qkv":
            kernels.qkv_rope(x, m.w_qkv_packed[l], sh.hq, sh.hkv, sh.head_dim, pos, m.freq, q, kv[0], kv[1], ws=ws)
        else:
            kernels.out_proj(x, m.w_o_packed[l], q.view(B, -1), ws=ws)


s = torch.cuda.Stream()
with torch.cuda.stream(s):
    run()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        run()
    for _ in range(3):
        g.replay()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    g.replay()
    e1.record(s)
    torch.cuda.synchronize()
    _lib.lib.rk_debug_proj_trace  # noqa
torch.cuda.synchronize()
print(f"graph of {sh.num_layers}: {e0.elapsed_time(e1) * 1000 / sh.num_layers:.2f} us per launch")
buf = (C.c_ulonglong * (148 * 16))()
assert _lib.lib.rk_debug_proj_trace(buf, 148 * 16) == 0
t = np.frombuffer(buf, dtype=np.uint64).reshape(148, 16).astype(np.int64)
t = t[t[:, 0] > 0]                               # CTAs of this launch (cluster grids use fewer than 148)
t0 = t[:, 0].min()
names = ["start", "1st W", "pdl done", "1st X", "last MMA", "epi done", "end", "last acc ld", "partial st",
         "ticket", "red loads", "finish"]
for i, nm in enumerate(names):
    ok = t[:, i] >= t0
    if not ok.any():
        continue
    col = (t[ok, i] - t0) / 1000.0
    print(f"{nm:11s} n {ok.sum():3d} min {col.min():7.2f}  p50 {np.median(col):7.2f}  max {col.max():7.2f} us")

ub = (C.c_ulonglong * 192)()
assert _lib.lib.rk_debug_proj_units(ub) == 0
u = (np.frombuffer(ub, dtype=np.uint64).reshape(3, 64).astype(np.int64) - t[0, 0]) / 1000.0
nu = int((u[0] > -1000).sum())
print("CTA 0 per unit (us from its start): wfull / x converted / hfull passed")
for i in range(min(nu, 24)):
    print(f"  {i:2d}  W {u[0, i]:6.2f}  Xconv {u[2, i]:6.2f}  MMA go {u[1, i]:6.2f}")
