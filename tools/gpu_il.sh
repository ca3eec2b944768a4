mkdir -p gpurun_out
exec > gpurun_out/il.log 2>&1
timeout 900 python -m pytest tests/test_gpu_proj.py tests/test_gpu_engine.py -q -x 2>&1 | tail -3
timeout 600 python tools/bench_token_step.py --batch 1 4 16 32 | cut -c1-260
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu --no-fetch-all --no-e2e | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['roofline']['frac'], d['roofline']['whole_step_frac'], d['roofline']['peak'])"
