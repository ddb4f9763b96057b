"""Summarise tools/ab_bench.sh output: pin result and words/s per variant."""
import glob
import json
import sys

for v in sys.argv[1:]:
    pin = open(f"gpurun_out/pin_{v}.log").read().strip().splitlines()[-2:]
    vals = []
    for f in sorted(glob.glob(f"gpurun_out/bench_{v}_*.log")):
        lines = [json.loads(x) for x in open(f) if x.startswith("{")]
        if lines:
            vals.append(round(lines[-1]["value"] / 1e6, 1))
    print(f"{v:14s} {' | '.join(pin)}  M words/s: {vals}")
