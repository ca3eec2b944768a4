mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_prefill.py -x -q 2>&1 | tail -3
timeout 300 python tools/bench_prefill.py --json gpurun_out/prefill_c3.json > gpurun_out/prefill_bench.log 2>&1
if [ "${PROF:-1}" = "1" ]; then
timeout 600 ncu --set full --clock-control none --import-source on -k regex:prefill_tc_kernel -s 2 -c 1 \
  -o gpurun_out/prefill_tc python tools/bench_prefill.py --nq 512 --reps 1 > gpurun_out/prefill_ncu.log 2>&1
fi
cat gpurun_out/prefill_bench.log; tail -2 gpurun_out/prefill_ncu.log
