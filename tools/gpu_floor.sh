# hot-row sink vs resident warps: sweep the warp floor over the configs[1] grid
mkdir -p gpurun_out
for f in 0 20 16 12 8; do
  SGNS_UPDATE_WARP_FLOOR=$f timeout 900 python bench.py --config micro --micro-grid --no-cpu-baseline > gpurun_out/floor_$f.log 2>&1
done
