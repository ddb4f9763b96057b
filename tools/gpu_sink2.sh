# asymmetric hot-row sinks (more M_in rows than M_out rows) on selected configs[1] shapes
mkdir -p gpurun_out
SH="65536,300,5,5;65536,300,2,5;65536,200,5,5;65536,200,2,5;65536,100,5,5;65536,100,10,5;65536,300,5,10;65536,300,5,15;65536,200,5,10;65536,200,10,5"
for h in auto 6,2 4,4 4,0 3,1 2,2; do
  if [ $h = auto ]; then unset SGNS_UPDATE_HOT; else export SGNS_UPDATE_HOT=$h; fi
  SGNS_UPDATE_DEBUG=1 timeout 900 python bench.py --config micro --micro-grid --micro-shape "$SH" --no-cpu-baseline --steps 10 > gpurun_out/sink2_${h/,/_}.log 2> gpurun_out/sink2_${h/,/_}.err
done
