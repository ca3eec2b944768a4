mkdir -p gpurun_out
exec > gpurun_out/pf2.log 2>&1
for pf in 0 1; do echo "RK_L2_PF=$pf"; RK_L2_PF=$pf timeout 600 python tools/bench_token_step.py --batch 1 4 16 | cut -c1-200; done
