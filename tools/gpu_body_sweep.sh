# configs[1] grid, K >= 10 shapes: launcher's choice vs forced F2G ("g") vs forced F2S ("s")
mkdir -p gpurun_out
SH=""
for d in 100 200 300; do for w in 2 5 10; do for k in 10 15; do SH="$SH;65536,$d,$w,$k"; done; done; done
SH=${SH#;}
for body in auto g s; do
  if [ $body = auto ]; then unset SGNS_UPDATE_BODY; else export SGNS_UPDATE_BODY=$body; fi
  timeout 900 python bench.py --config micro --micro-grid --micro-shape "$SH" --no-cpu-baseline > gpurun_out/body_$body.log 2>&1
done
