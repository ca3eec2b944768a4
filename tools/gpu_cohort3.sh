mkdir -p gpurun_out
exec > gpurun_out/cohort3.log 2>&1
timeout 600 python -m pytest tests/test_gpu_cohort.py -q 2>&1 | tail -3
for S in groups cohorts; do
  timeout 1200 python bench.py --workload c3 --serving $S --no-cpu --no-fetch-all --steps 3 --warmup 3 > gpurun_out/bench_c3_$S.json 2> gpurun_out/bench_c3_$S.err
  python -c "import json; d=json.loads(open('gpurun_out/bench_c3_$S.json').read().strip().splitlines()[-1]); r=d['roofline']; print('c3', '$S', round(d['value']), round(r['frac'],3), round(r['whole_step_frac'],3), round(d['e2e']['value']), d['breakdown_ms_group0'])" || tail -5 gpurun_out/bench_c3_$S.err
done
