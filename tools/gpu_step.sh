#!/bin/bash
# persistent whole-step kernel: parity tests, then the token-step microbench
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/step_smi.txt 2>&1
timeout 600 python -m pytest tests/test_gpu_step.py -x -q > gpurun_out/step_tests.log 2>&1
echo "tests exit $?" >> gpurun_out/step_tests.log
timeout 600 python tools/bench_step.py --workload c2 --batch 1 2 4 8 16 > gpurun_out/step_bench.log 2>&1
echo "bench exit $?" >> gpurun_out/step_bench.log
