timeout 600 python -m pytest tests/test_gpu_engine.py -x -q 2>&1 | tail -3
timeout 900 python bench.py --no-cpu > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; tail -2 gpurun_out/bench_c2.err; cat gpurun_out/bench_c2.json
