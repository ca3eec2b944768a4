# full GPU suite + smoke + memcheck/racecheck of the round-2 kernels + B=256 check
mkdir -p gpurun_out
exec > gpurun_out/full2.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
export PYTORCH_NO_CUDA_MEMORY_CACHING=1
timeout 1200 compute-sanitizer --tool memcheck --leak-check no --error-exitcode 99 --print-limit 20 \
  python -m pytest tests/test_gpu_decode_cluster.py tests/test_gpu_exact_scoring.py -q -x -k "f32 or pre or exact_scorer or unplanted" \
  > gpurun_out/san_mem2.log 2>&1; echo "memcheck rc=$?" >> gpurun_out/san_mem2.log
tail -3 gpurun_out/san_mem2.log
timeout 1200 compute-sanitizer --tool racecheck --racecheck-report hazard --error-exitcode 99 --print-limit 10 \
  python -m pytest tests/test_gpu_decode_cluster.py tests/test_gpu_exact_scoring.py -q -x -k "f32_vs_oracle and 2176 or exact_pre_scorer_matches_oracle and 4-28" \
  > gpurun_out/san_race2.log 2>&1; echo "racecheck rc=$?" >> gpurun_out/san_race2.log
tail -3 gpurun_out/san_race2.log
unset PYTORCH_NO_CUDA_MEMORY_CACHING
timeout 900 python bench.py --batch 256 --host-unique 16 --no-e2e --no-cpu --no-fetch-all --steps 2 --warmup 3 > gpurun_out/b256.json 2> gpurun_out/b256.err; echo "b256 rc=$?"
tail -3 gpurun_out/b256.err; cut -c1-300 gpurun_out/b256.json
