mkdir -p gpurun_out
exec > gpurun_out/r2l.log 2>&1
python -c "import __graft_entry__ as g; g.build()"
SRC=proj bash tools/build_variant.sh trace -DPJ_TRACE > /dev/null 2>&1 || echo trace build failed
for b in 1 16; do for w in qkv out; do echo "== B=$b $w"; ROUNDKV_B200_LIB=$PWD/variants_tmp/librk_trace.so timeout 120 python tools/proj_trace.py --batch $b --which $w 2>&1 | grep -v Warn; done; done
