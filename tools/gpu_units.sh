mkdir -p gpurun_out
exec > gpurun_out/units.log 2>&1
echo "== default"; python tools/bench_scoring.py --nq 512 | cut -c1-90
for u in 4 12 16 24; do echo "== RK_PREFILL_UNITS=$u balance 0"; RK_PREFILL_BALANCE=0 RK_PREFILL_UNITS=$u python tools/bench_scoring.py --nq 512 | cut -c1-90; done
echo "== prefill default"; python tools/bench_prefill.py 2>&1 | grep '"n_q": 512' | cut -c1-200
for u in 12 16; do echo "== prefill RK_PREFILL_UNITS=$u balance 0"; RK_PREFILL_BALANCE=0 RK_PREFILL_UNITS=$u python tools/bench_prefill.py 2>&1 | grep '"n_q": 512' | cut -c1-200; done
