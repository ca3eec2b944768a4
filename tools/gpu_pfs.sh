mkdir -p gpurun_out
exec > gpurun_out/pfs.log 2>&1
timeout 900 python -m pytest tests/test_gpu_selection_variants.py tests/test_gpu_prefill.py tests/test_gpu_fullsize.py tests/test_gpu_exact_scoring.py tests/test_gpu_engine.py -q -x 2>&1 | tail -15
timeout 600 python tools/bench_prefill.py 2>&1 | tail -3 | cut -c1-330
