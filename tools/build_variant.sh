#!/bin/bash
# Build an experimental librk variant with extra -D flags for some sources (default prefill_tc):
#   [SRC="decode_mma proj"] tools/build_variant.sh NAME -DFLAG ...  ->  variants_tmp/librk_NAME.so  (timing experiments)
name=$1; shift
d=build/variants/$name
rm -rf $d; mkdir -p $d variants_tmp
for f in paper_2502_15294_b200/csrc/*.cu; do b=$(basename $f .cu)
  if [[ " ${SRC:-prefill_tc} " == *" $b "* ]]; then
    nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr -Xcompiler -fPIC -Iinclude "$@" -c $f -o $d/$b.o || exit 1
  else cp build/librk/$b.o $d/$b.o; fi
done
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o variants_tmp/librk_$name.so $d/*.o -lcudart_static -lrt -ldl -lpthread
