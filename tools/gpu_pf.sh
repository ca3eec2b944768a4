mkdir -p gpurun_out
exec > gpurun_out/pf.log 2>&1
for pf in 0 1; do echo "RK_L2_PREFETCH=$pf"; RK_L2_PREFETCH=$pf timeout 600 python tools/bench_token_step.py --batch 1 4 16 32 | cut -c1-200; done
for pf in 0 1; do echo "bench RK_L2_PREFETCH=$pf"; RK_L2_PREFETCH=$pf timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu --no-fetch-all --no-e2e | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['roofline']['frac'], d['roofline']['whole_step_frac'])"; done
