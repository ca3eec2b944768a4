timeout 600 python -m pytest tests/test_gpu_engine.py -x -q 2>&1 | tail -15
timeout 600 python bench.py --workload c3 --steps 3 --warmup 3 --no-cpu > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err; tail -3 gpurun_out/bench_c3.err; cat gpurun_out/bench_c3.json
