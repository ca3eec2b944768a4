mkdir -p gpurun_out
exec > gpurun_out/r2n.log 2>&1
python -c "import __graft_entry__ as g; g.build()"
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_turn_c2_b16.csv python tools/profile_engine.py --eager --turns 1 --batch 16 --decode-steps 4 --profile-turns > gpurun_out/launches_turn.log 2>&1; echo "ncu list rc=$?"
python tools/traffic_summary.py gpurun_out/launches_turn_c2_b16.csv --batch 16 --decode-steps 4 --out gpurun_out/traffic_c2_tokenstep.json | tail -8
bash tools/sweep_c5.sh > gpurun_out/c5_sweep.jsonl; cat gpurun_out/c5_sweep.jsonl
