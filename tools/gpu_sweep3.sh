mkdir -p gpurun_out
BATCHES="1 2 4 8 16 32 64 128 256" bash tools/sweep_c5.sh > gpurun_out/c5_sweep3.jsonl 2> gpurun_out/c5_sweep3.err
timeout 1200 python bench.py --workload c3 --steps 3 --warmup 3 > gpurun_out/bench_c3e.json 2> gpurun_out/bench_c3e.err; echo "c3 rc=$?"
cut -c1-140 gpurun_out/c5_sweep3.jsonl
python -c "
import json; d=json.loads(open('gpurun_out/bench_c3e.json').read().strip().splitlines()[-1]); r=d['roofline']; print(d['value'], r['frac'], r['whole_step_frac'], d['e2e']['value'], d['config']['workload'][-120:])"
