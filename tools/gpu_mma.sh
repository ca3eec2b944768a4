mkdir -p gpurun_out
exec > gpurun_out/mma.log 2>&1
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_decode_cluster.py tests/test_gpu_engine.py tests/test_gpu_fullsize.py tests/test_gpu_selection_variants.py -q -x 2>&1 | tail -5
RK_DECODE_CLUSTER=0 timeout 600 python tools/bench_decode_layer.py --batches 1,16,32,64 --keys 2177,16513
RK_DECODE_CLUSTER=0 timeout 600 ncu --metrics l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum,gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:decode_mma -c 2 python tools/bench_decode_layer.py --batches 16 --keys 16513 --calls 2 2>&1 | grep -E "decode_mma|bank|duration|dram" | head -12
