# ncu --set full of the round-2 kernels: fp32 cluster decode (B=16, 16.5 K keys) and the DMMA exact scorer (512 rows)
mkdir -p gpurun_out
exec > gpurun_out/ncu2.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:decode_cluster -s 3 -c 1 -o gpurun_out/dc_f32_full \
  python tools/bench_decode_layer.py --batches 16 --keys 16513 --dtype f32 --calls 4 > /dev/null 2>&1; echo "ncu dc rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:exact_stats_dmma -s 2 -c 1 -o gpurun_out/dmma_full \
  python tools/bench_scoring.py --nq 512 --exact > /dev/null 2>&1; echo "ncu dmma rc=$?"
for f in dc_f32_full dmma_full; do
  ncu -i gpurun_out/$f.ncu-rep --page raw --csv > gpurun_out/$f.csv 2>/dev/null
done
ls -la gpurun_out/*.ncu-rep
