# Evidence at HEAD on one B200: GPU tests, smoke, default bench, reference arm, microbench (default selection + grid)
mkdir -p gpurun_out
timeout 600 python bench.py > gpurun_out/bench.log 2>&1; echo "rc=$?" >> gpurun_out/bench.log
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/gputest.log 2>&1; echo "rc=$?" >> gpurun_out/gputest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "rc=$?" >> gpurun_out/smoke.log
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref.log 2>&1; echo "rc=$?" >> gpurun_out/bench_ref.log
timeout 900 python bench.py --config micro > gpurun_out/micro.log 2>&1; echo "rc=$?" >> gpurun_out/micro.log
timeout 900 python bench.py --config micro --micro-grid --no-cpu-baseline > gpurun_out/micro_grid.log 2>&1; echo "rc=$?" >> gpurun_out/micro_grid.log
