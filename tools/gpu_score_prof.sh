#!/bin/bash
# scores-only scorer: per-role wait breakdown (PF_PROF variant) + one ncu --set full capture at n_q=512
mkdir -p gpurun_out
exec > gpurun_out/score_prof.log 2>&1
SRC=prefill_tc bash tools/build_variant.sh prof -DPF_PROF -lineinfo
echo "== PF_PROF scores-only"; ROUNDKV_B200_LIB=variants_tmp/librk_prof.so timeout 120 python tools/prefill_prof.py --score
echo "== PF_PROF attention"; ROUNDKV_B200_LIB=variants_tmp/librk_prof.so timeout 120 python tools/prefill_prof.py
echo "== bench"; timeout 300 python tools/bench_scoring.py | cut -c1-200
timeout 600 ncu --set full --clock-control none --import-source on -k regex:prefill_tc_kernel -s 2 -c 1 \
  -o gpurun_out/score_tc_r02 -f python tools/bench_scoring.py --nq 512 > gpurun_out/score_ncu.log 2>&1
tail -2 gpurun_out/score_ncu.log
