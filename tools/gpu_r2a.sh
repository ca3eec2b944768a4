mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_exact_scoring.py tests/test_gpu_selection_variants.py tests/test_gpu_reference_plugin.py tests/test_gpu_engine.py tests/test_gpu_pipeline.py -q -s -x > gpurun_out/r2a_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2a_pytest.log
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu > gpurun_out/r2a_bench.json 2> gpurun_out/r2a_bench.err; echo "bench rc=$?" >> gpurun_out/r2a_bench.err
tail -30 gpurun_out/r2a_pytest.log; cut -c1-600 gpurun_out/r2a_bench.json; tail -3 gpurun_out/r2a_bench.err
