# wide single-group body (d <= 128, K >= 8): parity, then d = 100 grid shapes vs the forced two-group body
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edges.py tests/test_gpu_fullsize.py -m gpu -q -p no:cacheprovider -x > gpurun_out/f2w_test.log 2>&1; echo "rc=$?" >> gpurun_out/f2w_test.log
SH=""
for w in 2 5 10; do for k in 10 15; do SH="$SH;65536,100,$w,$k"; done; done
SH=${SH#;}
for r in 1 2; do
for body in auto g; do
  if [ $body = auto ]; then unset SGNS_UPDATE_BODY; else export SGNS_UPDATE_BODY=$body; fi
  timeout 900 python bench.py --config micro --micro-grid --micro-shape "$SH" --no-cpu-baseline > gpurun_out/f2w_${body}_$r.log 2>&1
done; done
