# racecheck of one small tcgen05 prefill case with the hazard details
mkdir -p gpurun_out
timeout 1200 compute-sanitizer --tool racecheck --racecheck-report hazard --print-limit 40 \
  python -m pytest tests/test_gpu_prefill.py -q -x -k "16-1000" > gpurun_out/race_prefill.log 2>&1
echo "rc=$?" >> gpurun_out/race_prefill.log
grep -E "Error|Write|Read|at 0x|prefill_tc.cu|SUMMARY|passed|failed" gpurun_out/race_prefill.log | sort | uniq -c | sort -rn | head -40
