# round-2 refresh: full GPU suite, smoke, C2 bench (ours + reference arm), eager-turn launch list
mkdir -p gpurun_out
exec > gpurun_out/round2.log 2>&1
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc=$?"
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_turn_c2_b16.csv python tools/profile_engine.py --eager --turns 1 --batch 16 --decode-steps 4 --profile-turns > gpurun_out/launches_turn.log 2>&1; echo "ncu list rc=$?"
python tools/launch_summary.py gpurun_out/launches_turn_c2_b16.csv | head -12
python tools/traffic_summary.py gpurun_out/launches_turn_c2_b16.csv --batch 16 --decode-steps 4 --out gpurun_out/traffic_c2_tokenstep.json | tail -5
