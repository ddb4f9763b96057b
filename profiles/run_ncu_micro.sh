#!/bin/bash
# ncu evidence for the isolated minibatch kernel (configs[1] north-star shape d=300, w=5, K=5,
# 65,536 windows, snapshot mode, L2 flushed before every launch).  The plain command runs first.
set -e
CMD="python bench.py --config micro --micro-shape 65536,300,5,5 --steps 5 --warmup 3 --no-cpu-baseline"
mkdir -p gpurun_out
$CMD > gpurun_out/ncu_micro_plain.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:update_windows -s 3 -c 1 \
    -o gpurun_out/prof_micro $CMD > gpurun_out/ncu_micro_full.log 2>&1
