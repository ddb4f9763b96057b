mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/gputest.log 2>&1; echo "rc=$?" >> gpurun_out/gputest.log
timeout 900 python bench.py --config micro --no-cpu-baseline > gpurun_out/micro.log 2>&1
timeout 900 python tools/k_sweep.py 5 7 10 15 > gpurun_out/ksweep.log 2>&1
for r in 1 2; do timeout 300 python bench.py --steps 30 --no-cpu-baseline --no-e2e > gpurun_out/bench_$r.log 2>&1; done
