timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 300 python tools/bench_prefill.py --json gpurun_out/prefill_c3.json 2>&1 | cut -c1-250
timeout 900 python bench.py --workload c3 --steps 3 --warmup 3 --no-cpu > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err; tail -1 gpurun_out/bench_c3.err; python -c "import json; d=json.load(open('gpurun_out/bench_c3.json')); print(d['value'], d['roofline']['frac'], d['e2e']['value'], d['prefill'])"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:prefill_tc_kernel -s 2 -c 1 -o gpurun_out/prefill_tc python tools/bench_prefill.py --nq 512 --reps 1 > gpurun_out/prefill_ncu.log 2>&1; tail -1 gpurun_out/prefill_ncu.log
