mkdir -p gpurun_out
exec > gpurun_out/cohort2.log 2>&1
timeout 600 python -m pytest tests/test_gpu_cohort.py -q 2>&1 | tail -2
for N in 2 4; do
  timeout 900 python bench.py --batch 32 --serving cohorts --cohorts $N --no-cpu --no-fetch-all --steps 4 --warmup 3 > gpurun_out/bench_coh$N.json 2> gpurun_out/bench_coh$N.err
  python -c "import json; d=json.loads(open('gpurun_out/bench_coh$N.json').read().strip().splitlines()[-1]); r=d['roofline']; print($N, round(d['value']), round(r['frac'],3), round(r['whole_step_frac'],3), round(d['e2e']['value']), d['breakdown_ms_group0'])" || tail -5 gpurun_out/bench_coh$N.err
done
