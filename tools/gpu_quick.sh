# quick GPU check of selected test files: bash tools/gpu_quick.sh "<pytest args>"
mkdir -p gpurun_out
timeout 1200 python -m pytest $1 -q -x > gpurun_out/quick.log 2>&1; echo "rc=$?" >> gpurun_out/quick.log
tail -40 gpurun_out/quick.log
