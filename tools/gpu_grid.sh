# configs[1] grid: parity on all 27 shapes, then the microbench over the grid; default bench first (cold clock sampler check)
mkdir -p gpurun_out
timeout 600 python bench.py > gpurun_out/bench.log 2>&1; echo "rc=$?" >> gpurun_out/bench.log
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k "configs1_grid or snapshot" > gpurun_out/grid_test.log 2>&1; echo "rc=$?" >> gpurun_out/grid_test.log
timeout 1200 python bench.py --config micro --micro-grid --no-cpu-baseline > gpurun_out/micro_grid.log 2>&1; echo "rc=$?" >> gpurun_out/micro_grid.log
