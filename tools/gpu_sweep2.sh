# round-2 measurements: C5 sweep (B=1..256), C3 and C4 lines, default C2 line
mkdir -p gpurun_out
BATCHES="1 2 4 8 16 32 64 128 256" bash tools/sweep_c5.sh > gpurun_out/c5_sweep.jsonl 2> gpurun_out/c5_sweep.err
timeout 1200 python bench.py --workload c3 --steps 3 --warmup 3 > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err; echo "c3 rc=$?"
timeout 1200 python bench.py --workload c4 --steps 3 --warmup 3 --no-cpu > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; echo "c4 rc=$?"
cat gpurun_out/c5_sweep.jsonl | cut -c1-160
cut -c1-400 gpurun_out/bench_c3.json; cut -c1-400 gpurun_out/bench_c4.json
