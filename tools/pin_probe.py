"""Diagnostic: per-sentence oracle pin budget of the dynamic drivers over a grid of
shapes (tests/test_gpu_fast_pin.py protocol), printed as one line per case."""
import itertools
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import test_gpu_fast_pin as T  # noqa: E402


def main():
    import torch
    torch.cuda.set_device(0)
    dims = [int(x) for x in os.environ.get("PROBE_D", "4,8,16,32,64,100").split(",")]
    ks = [int(x) for x in os.environ.get("PROBE_K", "5").split(",")]
    vs = [int(x) for x in os.environ.get("PROBE_V", "12,5000").split(",")]
    ws = [int(x) for x in os.environ.get("PROBE_W", "5").split(",")]
    for kern in os.environ.get("PROBE_KERNELS", "ring,pipe").split(","):
        os.environ["SGNS_FAST_KERNEL"] = kern
        for d, k, v, w in itertools.product(dims, ks, vs, ws):
            t = T._pin_case(d, k, 16, window=w, V=v)
            print(kern, f"d={d} k={k} V={v} w={w}", {x: (round(y, 3) if isinstance(y, float) else y)
                                                      for x, y in t.items()}, flush=True)


if __name__ == "__main__":
    main()
