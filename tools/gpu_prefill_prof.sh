mkdir -p gpurun_out
timeout 300 python tools/bench_prefill.py --json gpurun_out/prefill_c3.json > gpurun_out/prefill_bench.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:prefill_tc_kernel -s 2 -c 1 \
  -o gpurun_out/prefill_tc python tools/bench_prefill.py --nq 512 --reps 1 > gpurun_out/prefill_ncu.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:score_tc_kernel -s 2 -c 1 \
  -o gpurun_out/score_tc python tools/bench_prefill.py --nq 512 --reps 1 > gpurun_out/score_ncu.log 2>&1
cat gpurun_out/prefill_bench.log; tail -1 gpurun_out/prefill_ncu.log gpurun_out/score_ncu.log
