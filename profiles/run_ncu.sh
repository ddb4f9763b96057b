#!/bin/bash
# ncu evidence for the fused driver kernel (run under gpurun on one B200).
# The plain command runs first and must exit 0 before ncu touches it.
set -e
CMD="python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline"
mkdir -p gpurun_out
$CMD > gpurun_out/ncu_plain.log 2>&1
# 1) launch list: every kernel with its device time (cold, serialised: compare shares)
#    (the cap covers the ~450 torch launches of the synthetic-corpus generator that run
#    before the timed region, then every launch of the warm-up and timed steps)
ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv \
    --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launches.log 2>&1
# 2) full set on one warm drive_kernel launch (skip the 3 warm-up launches)
ncu --set full --clock-control none --import-source on -k regex:drive_ -s 3 -c 1 \
    -o gpurun_out/prof_drive $CMD > gpurun_out/ncu_full.log 2>&1
