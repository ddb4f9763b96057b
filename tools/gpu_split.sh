# snapshot-mode input chunking for long windows: parity, then w = 10 shapes with the split off / auto / forced on
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edges.py -m gpu -q -p no:cacheprovider -x > gpurun_out/split_test.log 2>&1; echo "rc=$?" >> gpurun_out/split_test.log
SGNS_UPDATE_SPLIT=1 timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -x -k "snapshot or process_batch" > gpurun_out/split_test_forced.log 2>&1; echo "rc=$?" >> gpurun_out/split_test_forced.log
SH=""
for d in 100 200 300; do for k in 5 10 15; do SH="$SH;65536,$d,10,$k"; done; done
SH=${SH#;}
for m in 0 auto 1; do
  if [ $m = auto ]; then unset SGNS_UPDATE_SPLIT; else export SGNS_UPDATE_SPLIT=$m; fi
  SGNS_UPDATE_DEBUG=1 timeout 900 python bench.py --config micro --micro-grid --micro-shape "$SH" --no-cpu-baseline > gpurun_out/split_$m.log 2> gpurun_out/split_$m.err
done
