"""Per-role barrier-wait breakdown of prefill_tc_kernel (PF_PROF variant).
    ROUNDKV_B200_LIB=variants_tmp/librk_prof.so python tools/prefill_prof.py"""
import ctypes as C
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2502_15294_b200 import _lib, kernels, stats  # noqa: E402

SCORE = "--score" in sys.argv     # the scores-only form (multi-row watershed scorer)

hq, hkv, d, nq, R, T = 28, 4, 128, 512, 64, 1024
hist = R * T
s = hist + nq
k = torch.randn(s, hkv, d, device="cuda").bfloat16()
v = torch.randn(s, hkv, d, device="cuda").bfloat16()
q = torch.randn(nq, hq, d, device="cuda")
qp = torch.arange(hist, s, device="cuda")
kp = torch.arange(s, device="cuda")
bounds = [(r * T, (r + 1) * T, r) for r in range(R)] + [(hist, s, R)]


def run():
    if SCORE:
        stats.round_scores(q, k, qp, kp, bounds, R, chunk=1024, exact=False)
    else:
        kernels.prefill_attention(q, k, v, qp, kp)


for _ in range(3):
    run()
buf = (C.c_ulonglong * 64)()
_lib.lib.rk_pf_prof_read(buf)
run()
_lib.lib.rk_pf_prof_read(buf)
a = np.array(list(buf), dtype=np.float64).reshape(4, 16) / 148.0
names = {0: ["meta_full", "s_full", "buf_free(rescale)", "buf_free(unit end)", "pair bar"],
         1: ["q_full", "buf_free(QK)", "k_full", "p_full", "v_full"],
         2: ["k_empty", "q_empty"], 3: ["v_empty"]}
for role, rn in enumerate(["softmax w0", "MMA", "K producer", "V producer"]):
    tot = a[role, 15]
    parts = ", ".join(f"{n} {a[role, i] / tot * 100:.1f}%" for i, n in enumerate(names[role]))
    print(f"{rn:12s} total {tot:.0f} clk/CTA: {parts}")
