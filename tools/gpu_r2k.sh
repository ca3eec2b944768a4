mkdir -p gpurun_out
exec > gpurun_out/r2k.log 2>&1
python -c "import __graft_entry__ as g; g.build()"
timeout 300 python -m pytest tests/test_gpu_proj.py -q -x 2>&1 | tail -2
timeout 300 python tools/bench_token_step.py --batch 1 16 32 2>&1 | tail -3
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu --no-fetch-all --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('bench', d['value'], d['roofline']['frac'], d['roofline']['whole_step_frac'])"
SRC=proj bash tools/build_variant.sh trace -DPJ_TRACE > /dev/null 2>&1 || echo trace build failed
for b in 16; do for w in qkv out; do echo "== B=$b $w"; ROUNDKV_B200_LIB=$PWD/variants_tmp/librk_trace.so timeout 120 python tools/proj_trace.py --batch $b --which $w 2>&1 | grep -v "^  [ 0-9][0-9]  W"; done; done
