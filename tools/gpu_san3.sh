# compute-sanitizer over the round-2 engine paths (policies, fp32, HBM tier, cohorts)
mkdir -p gpurun_out
exec > gpurun_out/san3.log 2>&1
timeout 1500 compute-sanitizer --tool memcheck --leak-check no --error-exitcode 99 --print-limit 20 \
  python -m pytest tests/test_gpu_cohort.py tests/test_gpu_engine_policies.py -q -x -k "not drop or top_percent_drop-False" \
  > gpurun_out/san3_mem.log 2>&1; echo "memcheck rc=$?" >> gpurun_out/san3_mem.log
tail -4 gpurun_out/san3_mem.log
timeout 900 compute-sanitizer --tool synccheck --error-exitcode 99 --print-limit 10 \
  python -m pytest tests/test_gpu_cohort.py -q -x -k "row_masked" > gpurun_out/san3_sync.log 2>&1; echo "synccheck rc=$?" >> gpurun_out/san3_sync.log
tail -3 gpurun_out/san3_sync.log
