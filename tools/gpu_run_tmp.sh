mkdir -p gpurun_out
sed -n '/shared-memory hazards/,$p' tools/gpu_sanitize.sh | bash
