# A/B: pin tests at d=300/320 and the headline bench for each library variant given
mkdir -p gpurun_out
for v in "$@"; do
  export SGNS_LIB_OVERRIDE=$PWD/build_variants/$v.so
  timeout 600 python -m pytest tests/test_gpu_fast_pin.py -q -p no:cacheprovider -k "d300 or d320" > gpurun_out/pin_$v.log 2>&1
  echo "rc=$?" >> gpurun_out/pin_$v.log
  for rep in 1 2; do
    timeout 300 python bench.py --steps 30 --no-cpu-baseline --no-e2e > gpurun_out/bench_${v}_$rep.log 2>&1
  done
done
