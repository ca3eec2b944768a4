mkdir -p gpurun_out
exec > gpurun_out/fuse.log 2>&1
for B in 1 4 16; do for f in 0 1; do
  RK_FUSE_OUT_QKV=$f timeout 900 python bench.py --batch $B --no-e2e --no-cpu --no-fetch-all --steps 3 --warmup 3 2>gpurun_out/fuse_err.txt | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print($B, 'fuse=$f', round(d['value']), round(r['frac'],3), round(r['whole_step_frac'],3), d['breakdown_ms_group0']['decode'])" || tail -3 gpurun_out/fuse_err.txt
done; done
