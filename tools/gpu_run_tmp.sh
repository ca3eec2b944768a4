timeout 600 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_prefill.py tests/test_gpu_engine.py -x -q 2>&1 | tail -3
timeout 300 python tools/bench_prefill.py --json gpurun_out/prefill_c3.json 2>&1 | cut -c1-330
