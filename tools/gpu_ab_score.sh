#!/bin/bash
# A/B of the scores-only pass over librk variants (alternating, 2 reps), then the prefill / scoring parity tests
mkdir -p gpurun_out
exec > gpurun_out/ab_score.log 2>&1
for rep in 1 2; do
  for v in ${VARIANTS:-old new}; do
    if [ $v = new ]; then L=paper_2502_15294_b200/librk.so; else L=variants_tmp/librk_$v.so; fi
    echo "== $v"; ROUNDKV_B200_LIB=$L timeout 300 python tools/bench_scoring.py --nq 128,512,1024 | cut -c1-96
  done
done
echo "== prefill (new)"; timeout 300 python tools/bench_prefill.py --nq 512 | cut -c1-200
echo "== tests"
timeout 900 python -m pytest tests/test_gpu_prefill.py tests/test_gpu_selection_variants.py tests/test_gpu_fullsize.py tests/test_gpu_exact_scoring.py -q -x 2>&1 | tail -4
