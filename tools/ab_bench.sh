# A/B: pin tests at d=300/320 for each library variant, then the headline bench with the
# variants interleaved (rounds of one run each) so box drift hits all of them alike
mkdir -p gpurun_out
REPS=${REPS:-2}
for v in "$@"; do
  SGNS_LIB_OVERRIDE=$PWD/build_variants/$v.so timeout 600 python -m pytest tests/test_gpu_fast_pin.py -q -p no:cacheprovider -k "d300 or d320" > gpurun_out/pin_$v.log 2>&1
  echo "rc=$?" >> gpurun_out/pin_$v.log
done
for rep in $(seq 1 $REPS); do
  for v in "$@"; do
    SGNS_LIB_OVERRIDE=$PWD/build_variants/$v.so timeout 300 python bench.py --steps 30 --no-cpu-baseline --no-e2e > gpurun_out/bench_${v}_$rep.log 2>&1
  done
done
