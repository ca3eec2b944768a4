mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_prefill.py -x -q > gpurun_out/prefill_tests.log 2>&1; echo "rc=$?" >> gpurun_out/prefill_tests.log
tail -30 gpurun_out/prefill_tests.log
