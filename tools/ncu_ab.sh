set -x
mkdir -p gpurun_out
export SGNS_LIB_OVERRIDE=$PWD/build_variants/ns5.so
CMD="python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline"
timeout 300 python bench.py --steps 20 --no-cpu-baseline --no-e2e > gpurun_out/bench_ring.log 2>&1
timeout 300 $CMD > gpurun_out/plain.log 2>&1 || exit 1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:drive_ -s 3 -c 1 -o gpurun_out/prof_ring $CMD > gpurun_out/ncu_ring.log 2>&1
SGNS_FAST_KERNEL=pipe timeout 600 ncu --set full --clock-control none --import-source on -k regex:drive_ -s 3 -c 1 -o gpurun_out/prof_pipe $CMD > gpurun_out/ncu_pipe.log 2>&1
