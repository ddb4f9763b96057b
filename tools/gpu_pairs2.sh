# warp-pair driver with one staged-row area per pair (more resident pairs): pin tests, K sweep
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_fast_pin.py tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -x > gpurun_out/pairs_test.log 2>&1; echo "rc=$?" >> gpurun_out/pairs_test.log
timeout 900 python tools/k_sweep.py 5 8 10 13 15 > gpurun_out/pairs_ksweep.log 2>&1
