# variant comparison: token step (one group) + quick bench (two groups)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
SRC=proj bash tools/build_variant.sh b150 -DPJ_BUDGET_KB=150 > /dev/null 2>&1 || echo build fail b150
SRC="proj decode_cluster" bash tools/build_variant.sh co96 -DPJ_BUDGET_KB=96 -DRK_CL_STAGES=2 > /dev/null 2>&1 || echo build fail co96
SRC="decode_cluster" bash tools/build_variant.sh cl2 -DRK_CL_STAGES=2 > /dev/null 2>&1 || echo build fail cl2
exec > gpurun_out/r2j.log 2>&1
for v in base b150 co96 cl2; do
  if [ $v = base ]; then L=paper_2502_15294_b200/librk.so; else L=variants_tmp/librk_$v.so; fi
  echo "== $v"
  ROUNDKV_B200_LIB=$PWD/$L timeout 300 python tools/bench_token_step.py --batch 1 16 2>&1 | tail -2
  ROUNDKV_B200_LIB=$PWD/$L timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu --no-fetch-all --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('bench', d['value'], d['roofline']['frac'], d['roofline']['whole_step_frac'])"
done
