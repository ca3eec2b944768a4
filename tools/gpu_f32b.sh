mkdir -p gpurun_out
exec > gpurun_out/f32b.log 2>&1
timeout 900 python -m pytest tests/test_gpu_engine_policies.py tests/test_gpu_decode_cluster.py tests/test_gpu_proj.py tests/test_gpu_engine.py -q -x 2>&1 | tail -15
timeout 900 python bench.py --kv-dtype f32 --host-unique 8 --steps 3 --warmup 3 --no-cpu --no-fetch-all > gpurun_out/bench_f32.json 2> gpurun_out/bench_f32.err; echo "bench f32 rc=$?"
cut -c1-1500 gpurun_out/bench_f32.json; tail -3 gpurun_out/bench_f32.err
