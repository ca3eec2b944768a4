mkdir -p gpurun_out
exec > gpurun_out/ptrace2.log 2>&1
SRC=proj bash tools/build_variant.sh trace -DPJ_TRACE
for b in 1 16; do
echo "== qkv B=$b cluster"; ROUNDKV_B200_LIB=variants_tmp/librk_trace.so python tools/proj_trace.py --batch $b --which qkv | head -9
echo "== qkv B=$b ticketed (148 SMs)"; RK_PROJ_NO_CLUSTER=1 ROUNDKV_B200_LIB=variants_tmp/librk_trace.so python tools/proj_trace.py --batch $b --which qkv | head -14
done
for pf in 0 1; do echo "token step RK_PROJ_NO_CLUSTER=$pf"; if [ $pf = 1 ]; then export RK_PROJ_NO_CLUSTER=1; fi; timeout 600 python tools/bench_token_step.py --batch 1 16 | cut -c1-220; done
