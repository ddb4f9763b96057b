mkdir -p gpurun_out
for h in auto 2,2; do
  if [ $h = auto ]; then unset SGNS_UPDATE_HOT; else export SGNS_UPDATE_HOT=$h; fi
  SGNS_UPDATE_DEBUG=1 timeout 600 python bench.py --config micro --micro-shape "4096,300,5,5;16384,300,5,5" --no-cpu-baseline > gpurun_out/small_${h/,/_}.log 2> gpurun_out/small_${h/,/_}.err
done
