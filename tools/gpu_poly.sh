mkdir -p gpurun_out
exec > gpurun_out/poly.log 2>&1
for v in 0 2 3 4; do SRC=prefill_tc bash tools/build_variant.sh poly$v -DPF_POLY_OF8_SCORE=$v; done
echo "== default (1 of 8)"; python tools/bench_scoring.py | cut -c1-110
for v in 0 2 3 4; do echo "== poly $v of 8"; ROUNDKV_B200_LIB=variants_tmp/librk_poly$v.so python tools/bench_scoring.py | cut -c1-110; done
