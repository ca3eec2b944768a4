timeout 1200 python bench.py --workload c4 --steps 2 --warmup 3 --no-cpu > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; tail -1 gpurun_out/bench_c4.err
timeout 900 python bench.py --workload c3 --steps 3 --warmup 3 --no-cpu > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err; tail -1 gpurun_out/bench_c3.err
for f in c4 c3; do python -c "
import json; d=json.load(open('gpurun_out/bench_$f.json')); print('$f', round(d['value']), round(d['roofline']['frac'],3), round(d['roofline']['whole_step_frac'],3), round(d['e2e']['value']), d['gpu_kv_saved']['saved_frac'], d['h2d']['GBps'], d.get('prefill',{}).get('lower_layers_tflops_group0'))"; done
