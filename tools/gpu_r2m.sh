mkdir -p gpurun_out
exec > gpurun_out/r2m.log 2>&1
python -c "import __graft_entry__ as g; g.build()"
timeout 300 python -m pytest tests/test_gpu_proj.py -q -x 2>&1 | tail -2
for env in "" "RK_PROJ_FORCE_CLUSTER=1"; do
echo "== env $env"
env $env timeout 300 python tools/bench_token_step.py --batch 1 16 2>&1 | tail -2
env $env timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu --no-fetch-all --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('bench', d['value'], d['roofline']['frac'], d['roofline']['whole_step_frac'])"
done
