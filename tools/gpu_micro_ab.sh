# large-K update bodies: launcher choice vs forced F2G / F2S on the configs[1] large-K shapes;
# plus the static driver's K sweep after the register-budget change
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edges.py -q -p no:cacheprovider > gpurun_out/t_par.log 2>&1; echo "rc=$?" >> gpurun_out/t_par.log
S="65536,300,5,10;65536,300,5,15;65536,100,10,15"
for b in auto g s; do
  if [ $b = auto ]; then unset SGNS_UPDATE_BODY; else export SGNS_UPDATE_BODY=$b; fi
  timeout 600 python bench.py --config micro --no-cpu-baseline --micro-shape "$S" > gpurun_out/micro_body_$b.log 2>&1
done
unset SGNS_UPDATE_BODY
timeout 900 python tools/k_sweep.py --both 10 15 > gpurun_out/ksweep2.log 2>&1
