for a in "--question-noise 0.3" "--question-noise 1.0" "--question-noise 1.0 --no-round-cache"; do
timeout 600 python bench.py --no-cpu $a 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); h=d['h2d']
print(json.dumps({'args': '$a', 'value': round(d['value']), 'e2e': round(d['e2e']['value']), 'frac': round(d['roofline']['frac'],3), 'whole': round(d['roofline']['whole_step_frac'],3), 'h2d_GB_turn': round(h['bytes_per_turn_all_groups']/1e9,2), 'fetched': h['round_cache']['rounds_fetched_group0_last_turn'], 'kept': h['round_cache']['rounds_kept_group0']}))"
done | tee gpurun_out/round_cache_sweep.jsonl
