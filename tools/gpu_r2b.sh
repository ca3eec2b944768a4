mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_engine.py -q -x -s > gpurun_out/r2b_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2b_pytest.log
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu > gpurun_out/r2b_bench.json 2> gpurun_out/r2b_bench.err; echo "bench rc=$?" >> gpurun_out/r2b_bench.err
tail -40 gpurun_out/r2b_pytest.log; cut -c1-1500 gpurun_out/r2b_bench.json; tail -5 gpurun_out/r2b_bench.err
