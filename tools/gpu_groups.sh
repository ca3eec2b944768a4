mkdir -p gpurun_out
exec > gpurun_out/groups.log 2>&1
for B in 2 4 8 16; do for G in 1 2; do
  timeout 900 python bench.py --batch $B --groups $G --no-e2e --no-cpu --no-fetch-all --steps 3 --warmup 3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print($B, $G, round(d['value']), round(r['frac'],3), round(r['whole_step_frac'],3))"
done; done
