# warp-pair driver, K + 1 = 14 / 16 (7-8 output rows per warp): register cap 168 (12 warps/SM) vs 144 (14) vs 128 (16)
mkdir -p gpurun_out
for r in 1 2; do
for v in base wide144 wide128; do
  if [ $v = base ]; then unset SGNS_LIB_OVERRIDE; else export SGNS_LIB_OVERRIDE=$PWD/build_variants/$v.so; fi
  timeout 900 python tools/k_sweep.py 13 15 > gpurun_out/wide_${v}_$r.log 2>&1
done; done
