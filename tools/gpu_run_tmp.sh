timeout 300 python -m pytest tests/test_gpu_prefill.py tests/test_gpu_kernels.py -x -q -k "prefill or round_scores" 2>&1 | tail -2
for v in poly0 poly1 base poly3 poly4; do
  if [ $v = base ]; then lib=paper_2502_15294_b200/librk.so; else lib=variants_tmp/librk_$v.so; fi
  echo "== $v"; ROUNDKV_B200_LIB=$PWD/$lib timeout 120 python tools/bench_prefill.py --nq 512,1024 --reps 10 2>&1 | python -c "
import sys,json
for l in sys.stdin:
    if l.startswith('{'): d=json.loads(l); print(d['n_q'], round(d['ms_prefill'],4), round(d['ms_prefill_fused_scoring'],4), round(d['ms_separate_scorer'],4), round(d['algo_tflops']))"
done
