#!/bin/bash
# end-of-round refresh: GPU suite, smoke, C2/C3/C4 bench lines, reference arm, C2 launch list
mkdir -p gpurun_out/refresh
cd gpurun_out/refresh
R=$GRAFT_REPO_ROOT
timeout 1200 python -m pytest $R/tests -m gpu -q -p no:cacheprovider > pytest_gpu.log 2>&1; echo "pytest rc=$?" >> pytest_gpu.log
(cd $R && timeout 300 python -c "import __graft_entry__ as g; g.smoke()") > smoke.log 2>&1; echo "smoke rc=$?" >> smoke.log
timeout 900 python $R/bench.py > c2.json 2> c2.err
timeout 900 python $R/bench.py --workload c3 > c3.json 2> c3.err
timeout 900 python $R/bench.py --workload c4 > c4.json 2> c4.err
timeout 900 python $R/bench.py --impl reference > ref.json 2> ref.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s 1500 -c 3000 --csv --log-file launches_c2.csv \
  python $R/bench.py --steps 1 --warmup 1 --no-cpu --no-e2e --no-fetch-all --decode-steps 16 > launches.log 2>&1
