"""Per-kernel device-time shares from an ncu launch list.

Reads the `ncu --metrics gpu__time_duration.sum --csv --log-file X` output and prints,
for the launches from the first match of PATTERN on (the warm-up and timed steps), each
kernel's share of device time.  ncu times are cold and serialised: compare shares.

  python tools/launch_share.py gpurun_out/launches.csv [PATTERN]
"""
import csv
import sys
from collections import OrderedDict


def main(path, pattern="drive_"):
    with open(path) as fh:
        lines = [ln for ln in fh if ln.startswith('"')]
    rows = list(csv.DictReader(lines))
    launches = []
    for r in rows:
        if r["Metric Name"] != "gpu__time_duration.sum":
            continue
        v = float(r["Metric Value"])
        unit = r["Metric Unit"]
        ms = v / 1e6 if unit in ("nsecond", "ns") else v / 1e3 if unit in ("usecond", "us") else v if unit in ("msecond", "ms") else v * 1e3
        launches.append((r["Kernel Name"], ms))
    first = next((i for i, (n, _) in enumerate(launches) if pattern in n), None)
    print(f"total launches {len(launches)}")
    if first is None:
        print(f"no launch matches {pattern!r}")
        return
    hit = [l for l in launches[first:] if pattern in l[0]]
    before = launches[:first]
    print(f"first {pattern} launch index {first} count {len(hit)}")
    print(f"before it: {len(before)} launches, {sum(t for _, t in before):.2f} ms")
    tail = launches[first:]
    tot = sum(t for _, t in tail)
    print(f"from it on: {len(tail)} launches, {tot:.3f} ms")
    agg = OrderedDict()
    for n, t in tail:
        a = agg.setdefault(n, [0.0, 0])
        a[0] += t
        a[1] += 1
    for n, (t, c) in sorted(agg.items(), key=lambda kv: -kv[1][0]):
        print(f"  {100 * t / tot:6.2f}%  {t:9.3f} ms  x {c:3d}  mean {t / c:.3f} ms  {n[:110]}")


if __name__ == "__main__":
    main(*sys.argv[1:])
