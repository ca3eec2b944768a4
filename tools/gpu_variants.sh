# Time tools/bench_prefill.py (C3, n_q=512) with librk variants built by tools/build_variant.sh
for v in ${VARIANTS:-base}; do
  if [ $v = base ]; then lib=paper_2502_15294_b200/librk.so; else lib=variants_tmp/librk_$v.so; fi
  echo "== $v"; ROUNDKV_B200_LIB=$PWD/$lib timeout 120 python tools/bench_prefill.py --nq 512 --reps 5 2>&1 | tail -1 | cut -c1-160
done
