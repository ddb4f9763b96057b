# Diagnostic: the production kernel at d = 300 (partial last slot) vs d = 320 / 256 (whole slots), interleaved.
mkdir -p gpurun_out
timeout 600 python bench.py > gpurun_out/bench.log 2>&1; echo "rc=$?" >> gpurun_out/bench.log
for r in 1 2; do for d in 300 320 256; do
  SGNS_BENCH_DIM=$d timeout 300 python bench.py --steps 30 --no-cpu-baseline --no-e2e > gpurun_out/dim_${d}_$r.log 2>&1
done; done
