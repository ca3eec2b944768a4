#!/bin/bash
# which side bounds the scores-only pass: no exp2 (MMA + pipeline only) vs one MMA per tile (softmax only)
mkdir -p gpurun_out
exec > gpurun_out/score_bound.log 2>&1
SRC=prefill_tc bash tools/build_variant.sh noexp -DPF_EXP_OFF 2>/dev/null
SRC=prefill_tc bash tools/build_variant.sh mmaone -DPF_MMA_ONE 2>/dev/null
for v in default noexp mmaone; do
  echo "== $v"
  if [ $v = default ]; then L=paper_2502_15294_b200/librk.so; else L=variants_tmp/librk_$v.so; fi
  ROUNDKV_B200_LIB=$L timeout 300 python tools/bench_scoring.py --nq 512,1024 | cut -c1-90
  ROUNDKV_B200_LIB=$L timeout 300 ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_elapsed -k regex:prefill_tc_kernel -s 2 -c 1 python tools/bench_scoring.py --nq 512 2>&1 | grep -E "duration|tensor|xu"
done
