mkdir -p gpurun_out
exec > gpurun_out/budget.log 2>&1
for kb in 100 120; do SRC=proj bash tools/build_variant.sh b$kb -DPJ_BUDGET_KB=$kb; done
for v in default b100 b120; do
  if [ $v = default ]; then unset ROUNDKV_B200_LIB; else export ROUNDKV_B200_LIB=variants_tmp/librk_$v.so; fi
  echo "== $v"; timeout 600 python tools/bench_token_step.py --batch 1 4 16 | cut -c1-150
done
for v in default b100; do
  if [ $v = default ]; then unset ROUNDKV_B200_LIB; else export ROUNDKV_B200_LIB=variants_tmp/librk_$v.so; fi
  echo "== bench $v"; timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu --no-fetch-all --no-e2e | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['roofline']['frac'])"
done
