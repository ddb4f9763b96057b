# update kernel: L2 prefetch of the warp's next window on / off (Zipf grid subset + uniform ids), after parity
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edges.py -m gpu -q -p no:cacheprovider -x > gpurun_out/pf_test.log 2>&1; echo "rc=$?" >> gpurun_out/pf_test.log
for r in 1 2; do for pf in 1 0; do
  SGNS_UPDATE_PREFETCH=$pf timeout 900 python bench.py --config micro --micro-grid --no-cpu-baseline --steps 10 > gpurun_out/pf_${pf}_$r.log 2>&1
done; done
for pf in 1 0; do
  SGNS_UPDATE_PREFETCH=$pf timeout 900 python bench.py --config micro --micro-ids uniform --no-cpu-baseline > gpurun_out/pf_uni_$pf.log 2>&1
  SGNS_UPDATE_PREFETCH=$pf timeout 900 python bench.py --config micro --no-cpu-baseline > gpurun_out/pf_sel_$pf.log 2>&1
done
