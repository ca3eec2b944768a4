mkdir -p gpurun_out
exec > gpurun_out/split.log 2>&1
timeout 900 python -m pytest tests/test_gpu_decode_cluster.py tests/test_gpu_kernels.py tests/test_gpu_engine.py -q -x 2>&1 | tail -3
for sp in 0 1; do echo "RK_DECODE_SPLIT=$sp"; RK_DECODE_SPLIT=$sp timeout 600 python tools/bench_decode_layer.py --batches 1,2 --keys 16513,65537 | cut -c1-130; done
for sp in 0 1; do echo "bench B=1 RK_DECODE_SPLIT=$sp"; RK_DECODE_SPLIT=$sp timeout 600 python bench.py --batch 1 --no-e2e --no-cpu --no-fetch-all --steps 3 --warmup 3 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), round(d['roofline']['frac'],3))"; done
