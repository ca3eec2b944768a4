#!/bin/bash
# cohort serving vs the default groups at small / mid batches (C2 shapes), same box, alternating
mkdir -p gpurun_out
exec > gpurun_out/cohort_small.jsonl 2> gpurun_out/cohort_small.err
for B in 8 16 32; do
  for mode in groups cohorts; do
    timeout 900 python bench.py --batch $B --serving $mode --no-cpu --no-fetch-all --steps 3 --warmup 3 |
      python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline']; print(json.dumps(dict(batch=$B, serving='$mode', tok_s=d['value'], e2e=d['e2e']['value'], frac=r['frac'], whole=r.get('whole_step_frac'), clocks=d['clocks'])))"
  done
done
