# compute-sanitizer memcheck over the small-shape GPU parity tests
mkdir -p gpurun_out
export PYTORCH_NO_CUDA_MEMORY_CACHING=1
timeout 1500 compute-sanitizer --tool memcheck --leak-check no --error-exitcode 99 --print-limit 20 \
  python -m pytest tests/test_gpu_kernels.py tests/test_gpu_prefill.py -q -x -k "not 513 and not 512" \
  > gpurun_out/sanitize_memcheck.log 2>&1; echo "memcheck rc=$?" >> gpurun_out/sanitize_memcheck.log
# (graph capture needs torch's caching allocator: no PYTORCH_NO_CUDA_MEMORY_CACHING here)
env -u PYTORCH_NO_CUDA_MEMORY_CACHING timeout 900 compute-sanitizer --tool memcheck --leak-check no --error-exitcode 99 --print-limit 20 \
  python -m pytest tests/test_gpu_engine.py tests/test_gpu_pipeline.py tests/test_gpu_calibration.py -q -x -k "not accounting" \
  > gpurun_out/sanitize_memcheck_engine.log 2>&1; echo "memcheck rc=$?" >> gpurun_out/sanitize_memcheck_engine.log
tail -4 gpurun_out/sanitize_memcheck.log; tail -4 gpurun_out/sanitize_memcheck_engine.log
# shared-memory hazards / barrier misuse on the pipelined kernels (small shapes)
timeout 1200 compute-sanitizer --tool racecheck --racecheck-report hazard --error-exitcode 99 --print-limit 10 \
  python -m pytest tests/test_gpu_prefill.py tests/test_gpu_kernels.py -q -x -k "16-1000 or 64-0 or decode_append or fused_decode or peaked" \
  > gpurun_out/sanitize_racecheck.log 2>&1; echo "racecheck rc=$?" >> gpurun_out/sanitize_racecheck.log
timeout 1200 compute-sanitizer --tool synccheck --error-exitcode 99 --print-limit 10 \
  python -m pytest tests/test_gpu_prefill.py tests/test_gpu_kernels.py -q -x -k "16-1000 or 64-0 or decode_append or fused_decode or peaked" \
  > gpurun_out/sanitize_synccheck.log 2>&1; echo "synccheck rc=$?" >> gpurun_out/sanitize_synccheck.log
tail -3 gpurun_out/sanitize_racecheck.log; tail -3 gpurun_out/sanitize_synccheck.log
