#!/bin/bash
# compute-sanitizer memcheck / synccheck / racecheck of the persistent step kernel on the small parity configs
mkdir -p gpurun_out
export RK_STEP_PATIENCE_S=600
for tool in memcheck synccheck racecheck; do
  extra=""; [ $tool = memcheck ] && extra="--leak-check no"; [ $tool = racecheck ] && extra="--racecheck-report hazard"
  timeout 1500 compute-sanitizer --tool $tool $extra --kernel-name kns=step_kernel --error-exitcode 99 --print-limit 20 \
    python -m pytest tests/test_gpu_step.py -x -q -k "hidden_state or (layered_kernels and 4)" \
    > gpurun_out/step_san_$tool.log 2>&1
  echo "exit $?" >> gpurun_out/step_san_$tool.log
done
