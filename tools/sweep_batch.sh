# small-batch sweep of the C2 (or WORKLOAD=c4) turn (one dialogue group): decode tokens/s and the
# decode kernels' HBM fraction per batch; one JSON line per batch on stdout
for B in ${BATCHES:-1 2 4 8 16}; do
  timeout 900 python bench.py --workload ${WORKLOAD:-c2} --batch $B --groups 1 --no-e2e --no-cpu --steps ${STEPS:-3} --warmup 3 2>/dev/null |
    python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline']; print(json.dumps(dict(batch=$B, tok_s=d['value'], ms_step=d['ms_per_step'], frac=r['frac'], whole=r.get('whole_step_frac'), decode_path='${RK_DECODE_CLUSTER:-auto}', workload='${WORKLOAD:-c2}')))"
done
