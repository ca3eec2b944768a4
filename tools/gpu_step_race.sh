#!/bin/bash
# racecheck: the step kernel with the plain mbarrier wait loop, and decode_mma (bulk copies + ldmatrix) for comparison
mkdir -p gpurun_out
export RK_STEP_PATIENCE_S=600
ROUNDKV_B200_LIB=variants_tmp/librk_plainwait.so timeout 1500 compute-sanitizer --tool racecheck --racecheck-report hazard \
  --kernel-name kns=step_kernel --error-exitcode 99 --print-limit 4 \
  python -m pytest tests/test_gpu_step.py -x -q -k "hidden_state" > gpurun_out/step_race_plain.log 2>&1
echo "exit $?" >> gpurun_out/step_race_plain.log
timeout 1500 compute-sanitizer --tool racecheck --racecheck-report hazard --kernel-name kns=decode_mma \
  --error-exitcode 99 --print-limit 4 \
  python -m pytest tests/test_gpu_kernels.py -x -q -k "fused_decode" > gpurun_out/mma_race.log 2>&1
echo "exit $?" >> gpurun_out/mma_race.log
