# A/B of the warp-pair driver (K + 1 = 9..16): the pair pin tests for each library variant, then
# the production K sweep (K = 10, 15) with the variants interleaved
mkdir -p gpurun_out
REPS=${REPS:-2}
for v in "$@"; do
  SGNS_LIB_OVERRIDE=$PWD/build_variants/$v.so timeout 900 python -m pytest tests/test_gpu_fast_pin.py -q -p no:cacheprovider -k "k8_ or k9_ or k10_ or k11_ or k12_ or k14_ or k15_" > gpurun_out/ppin_$v.log 2>&1
  echo "rc=$?" >> gpurun_out/ppin_$v.log
done
for rep in $(seq 1 $REPS); do
  for v in "$@"; do
    SGNS_LIB_OVERRIDE=$PWD/build_variants/$v.so timeout 600 python tools/k_sweep.py 10 15 > gpurun_out/ksw_${v}_$rep.log 2>&1
  done
done
for v in "$@"; do
  echo "$v: $(tail -n 2 gpurun_out/ppin_$v.log | tr '\n' ' ')"
  for rep in $(seq 1 $REPS); do grep -o '"K": [0-9]*, "schedule": "auto", "words_per_sec": [0-9.]*' gpurun_out/ksw_${v}_$rep.log | tr '\n' ' '; echo; done
done
