"""Summarise an ncu report: headline metrics + top stall reasons / instructions.

    python tools/ncu_stalls.py gpurun_out/x.ncu-rep [--top 25]
"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[sys.argv.index("--top") + 1]) if "--top" in sys.argv else 25
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, vals = rows[0], rows[2]
want = ["gpu__time_duration.sum", "sm__pipe_tensor_cycles_active.avg.pct", "tensor_op_utchmma_src_bf16_dst_fp32_sparsity_off.avg.pct_of_peak_sustained_elapsed",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "sm__issue_active.avg.pct",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__dram_throughput.avg.pct", "launch__registers_per_thread",
        "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "sm__cycles_elapsed.avg"]
for h, v in zip(hdr, vals):
    if any(w in h for w in want) and "per_second" not in h and ".max" not in h and ".min" not in h:
        print(f"{h:90s} {v}")
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
hdr, data = rows[1], rows[2:]
ix = {h: i for i, h in enumerate(hdr)}
S = "Warp Stall Sampling (All Samples)"
tot = sum(float(r[ix[S]] or 0) for r in data) or 1.0
cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
agg = {h: sum(float(r[ix[h]] or 0) for r in data) for h in cols}
print("stall reasons (% of samples):", ", ".join(f"{h[6:]} {100 * v / tot:.1f}" for h, v in
                                               sorted(agg.items(), key=lambda x: -x[1])[:8]))
for r in sorted(data, key=lambda r: -float(r[ix[S]] or 0))[:top]:
    main = max(cols, key=lambda h: float(r[ix[h]] or 0))
    print(f"{100 * float(r[ix[S]] or 0) / tot:5.2f}%  {main[6:]:18s} {r[ix['Source']][:90]}")
