mkdir -p gpurun_out
exec > gpurun_out/cohort.log 2>&1
timeout 600 python -m pytest tests/test_gpu_cohort.py -q 2>&1 | tail -2
for B in 32 64; do for S in groups cohorts; do
  timeout 900 python bench.py --batch $B --serving $S --no-cpu --no-fetch-all --steps 4 --warmup 3 $( [ $B = 64 ] && echo --host-unique 16 ) > gpurun_out/bench_${S}_$B.json 2> gpurun_out/bench_${S}_$B.err
  python -c "import json; d=json.loads(open('gpurun_out/bench_${S}_$B.json').read().strip().splitlines()[-1]); r=d['roofline']; print($B, '$S', round(d['value']), round(r['frac'],3), round(r['whole_step_frac'],3), round(d['e2e']['value']), d['breakdown_ms_group0'])" || tail -5 gpurun_out/bench_${S}_$B.err
done; done
for S in groups cohorts; do
  timeout 1200 python bench.py --workload c4 --serving $S --no-cpu --no-fetch-all --no-e2e --steps 3 --warmup 3 > gpurun_out/bench_c4_$S.json 2> gpurun_out/bench_c4_$S.err
  python -c "import json; d=json.loads(open('gpurun_out/bench_c4_$S.json').read().strip().splitlines()[-1]); r=d['roofline']; print('c4', '$S', round(d['value']), round(r['frac'],3), round(r['whole_step_frac'],3))" || tail -5 gpurun_out/bench_c4_$S.err
done
