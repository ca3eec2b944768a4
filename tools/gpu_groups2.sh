mkdir -p gpurun_out
exec > gpurun_out/groups2.log 2>&1
for W in c3 c4; do for G in 1 2; do
  timeout 1200 python bench.py --workload $W --groups $G --no-e2e --no-cpu --no-fetch-all --steps 3 --warmup 3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$W', $G, round(d['value']), round(r['frac'],3), round(r['whole_step_frac'],3))"
done; done
for G in 1 2; do timeout 900 python bench.py --batch 32 --groups $G --no-e2e --no-cpu --no-fetch-all --steps 3 --warmup 3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('c2-32', $G, round(d['value']), round(r['frac'],3), round(r['whole_step_frac'],3))"; done
