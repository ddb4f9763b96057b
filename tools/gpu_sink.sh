# hot-row sink size vs resident warps: force each sink candidate over the configs[1] grid
mkdir -p gpurun_out
for h in 8,8 4,4 2,2 1,1 0,1; do
  SGNS_UPDATE_DEBUG=1 SGNS_UPDATE_HOT=$h timeout 900 python bench.py --config micro --micro-grid --no-cpu-baseline --steps 10 > gpurun_out/sink_${h/,/_}.log 2> gpurun_out/sink_${h/,/_}.err
done
