# C5 batch sweep on one GPU (the per-GPU share of 1-256 dialogues over 1/2/4/8 GPUs) at C2 shapes:
# dialogues in bench.py's default groups (one below 32 dialogues, two from 32), the model on the GPU;
# one JSON line per batch on stdout
for B in ${BATCHES:-1 2 4 8 16 32 64 128 256}; do
  HU=0; if [ $B -ge 64 ]; then HU=16; fi
  timeout 1200 python bench.py --workload ${WORKLOAD:-c2} --batch $B --host-unique $HU --no-e2e --no-cpu --no-fetch-all --steps ${STEPS:-2} --warmup 3 2>/dev/null |
    python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline']; print(json.dumps(dict(batch=$B, host_unique=$HU, tok_s=d['value'], ms_step=d['ms_per_step'], frac=r['frac'], whole=r.get('whole_step_frac'), kernels=r['kernel'][r['kernel'].find('['):r['kernel'].find(']')+1], clocks=d['clocks'], workload='${WORKLOAD:-c2}')))" || echo "{\"batch\": $B, \"error\": true}"
done
