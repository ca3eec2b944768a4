timeout 300 python tools/bench_decode_layer.py --batches 1,4,16 2>&1 | tee gpurun_out/decode_layer_rk.jsonl
timeout 600 python tools/bench_flashinfer_decode.py --batches 1,4,16 2>&1 | tail -8 | tee gpurun_out/decode_layer_flashinfer.jsonl
