mkdir -p gpurun_out
exec > gpurun_out/f32.log 2>&1
timeout 900 python -m pytest tests/test_gpu_decode_cluster.py -q -x 2>&1 | tail -15
timeout 600 python tools/bench_decode_layer.py --batches 1,4,8,16 --keys 2177,16513 --dtype f32
timeout 600 python tools/bench_decode_layer.py --batches 1,4,8,16 --keys 2177,16513 --dtype bf16
