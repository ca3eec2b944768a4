#!/bin/bash
# last validation at HEAD: GPU suite, smoke, C2 line, then the C5 sweep B = 1..256
mkdir -p gpurun_out/final2
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/final2/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/final2/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final2/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/final2/smoke.log
timeout 900 python bench.py > gpurun_out/final2/c2.json 2> gpurun_out/final2/c2.err
BATCHES="1 2 4 8 16 32 64 128 256" bash tools/sweep_c5.sh > gpurun_out/final2/c5_sweep.jsonl 2> gpurun_out/final2/c5_sweep.err
