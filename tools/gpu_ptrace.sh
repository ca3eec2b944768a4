mkdir -p gpurun_out
exec > gpurun_out/ptrace.log 2>&1
SRC=proj bash tools/build_variant.sh trace -DPJ_TRACE
for w in qkv out; do for b in 1 16; do
ROUNDKV_B200_LIB=variants_tmp/librk_trace.so python tools/proj_trace.py --batch $b --which $w
done; done
