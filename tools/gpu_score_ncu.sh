#!/bin/bash
mkdir -p gpurun_out
exec > gpurun_out/score_ncu2.log 2>&1
SRC=prefill_tc bash tools/build_variant.sh mmaone -DPF_MMA_ONE -lineinfo 2>/dev/null
timeout 600 ncu --set full --clock-control none --import-source on -k regex:prefill_tc_kernel -s 2 -c 1 \
  -o gpurun_out/score_tc_parity -f python tools/bench_scoring.py --nq 512
ROUNDKV_B200_LIB=variants_tmp/librk_mmaone.so timeout 600 ncu --set full --clock-control none --import-source on -k regex:prefill_tc_kernel -s 2 -c 1 \
  -o gpurun_out/score_tc_mmaone -f python tools/bench_scoring.py --nq 512
