# round-end style GPU check: tests, smoke, benches (ours, reference, N=2 on one GPU), launch list + traffic, ncu captures
mkdir -p gpurun_out
exec > gpurun_out/round.log 2>&1
python -c "import __graft_entry__ as g; g.build()"
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
tail -2 gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc=$?"
RK_SHARE_GPU=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --batch 16 --host-unique 4 --steps 3 --warmup 3 --no-cpu --no-fetch-all > gpurun_out/bench_n2.json 2> gpurun_out/bench_n2.err; echo "n2 rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_turn_c2_b16.csv python tools/profile_engine.py --eager --turns 1 --batch 16 --decode-steps 4 > gpurun_out/launches_turn.log 2>&1; echo "ncu list rc=$?"
python tools/traffic_summary.py gpurun_out/launches_turn_c2_b16.csv --batch 16 --decode-steps 4 --out gpurun_out/traffic_c2_tokenstep.json | tail -5
timeout 600 ncu --set full --import-source on --clock-control none -k regex:proj_tc -s 40 -c 2 -o gpurun_out/proj_tc_full python tools/profile_engine.py --eager --turns 1 --batch 16 --decode-steps 2 > gpurun_out/ncu_proj.log 2>&1; echo "ncu proj rc=$?"
timeout 600 ncu --set full --import-source on --clock-control none -k regex:decode_cluster -s 40 -c 1 -o gpurun_out/decode_cluster_full python tools/profile_engine.py --eager --turns 1 --batch 16 --decode-steps 2 > gpurun_out/ncu_dc.log 2>&1; echo "ncu dc rc=$?"
