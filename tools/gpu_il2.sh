mkdir -p gpurun_out
exec > gpurun_out/il2.log 2>&1
for r in 1 2; do for il in 0 1; do
echo "RK_PROJ_INTERLEAVE=$il"; RK_PROJ_INTERLEAVE=$il timeout 900 python bench.py --steps 4 --warmup 3 --no-cpu --no-fetch-all --no-e2e | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['roofline']['frac'], d['roofline']['whole_step_frac'], d['roofline']['peak'])"
done; done
for il in 0 1; do RK_PROJ_INTERLEAVE=$il timeout 600 python tools/bench_token_step.py --batch 1 16 | cut -c1-120; done
