mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r2c_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2c_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2c_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/r2c_smoke.log
timeout 900 python bench.py > gpurun_out/r2c_bench.json 2> gpurun_out/r2c_bench.err; echo "bench rc=$?" >> gpurun_out/r2c_bench.err
tail -30 gpurun_out/r2c_pytest.log; tail -3 gpurun_out/r2c_smoke.log; cut -c1-2500 gpurun_out/r2c_bench.json; tail -5 gpurun_out/r2c_bench.err
