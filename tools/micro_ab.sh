# configs[1] microbench for each library variant (interleaved rounds) + the snapshot parity tests
mkdir -p gpurun_out
REPS=${REPS:-2}
for v in "$@"; do
  SGNS_LIB_OVERRIDE=$PWD/build_variants/$v.so timeout 900 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -k "snapshot or process_batch or disjoint" > gpurun_out/mpin_$v.log 2>&1
  echo "rc=$?" >> gpurun_out/mpin_$v.log
done
for rep in $(seq 1 $REPS); do
  for v in "$@"; do
    SGNS_LIB_OVERRIDE=$PWD/build_variants/$v.so timeout 900 python bench.py --config micro --no-cpu-baseline > gpurun_out/micro_${v}_$rep.log 2>&1
  done
done
