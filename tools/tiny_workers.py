"""Tiny config (BASELINE configs[0]) quality vs the number of concurrent device workers:
per-epoch loss (every cell scored) and planted-cluster rho of the production path against
the reference algorithm at threads=1 (oracle), mean of 3 seeds per worker count.

    python tools/tiny_workers.py 64 128 256 488 1024
"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def main(workers):
    import torch  # noqa: F401
    import test_gpu_e2e as E
    from paper_1604_04661_b200.synthetic import tiny_config_corpus
    syn = tiny_config_corpus(seed=0)
    ref = [E._reference_run(syn, s) for s in (1, 2, 3)]
    rl = float(np.mean([r[1] for r in ref]))
    rr = float(np.mean([E._rho(r[0], syn) for r in ref]))
    out = {"ref_loss": rl, "ref_rho": rr, "rows": []}
    for w in workers:
        runs = [E._gpu_run(syn, s, workers=w) for s in (1, 2, 3)]
        gl = float(np.mean([st.loss_by_epoch[0] for _, st in runs]))
        gr = float(np.mean([E._rho(v, syn) for v, _ in runs]))
        out["rows"].append({"workers": w, "loss": gl, "loss_rel": gl / rl - 1, "rho": gr, "rho_diff": gr - rr})
        print(json.dumps(out["rows"][-1]), flush=True)
    print(json.dumps(out))


if __name__ == "__main__":
    main([int(x) for x in sys.argv[1:]] or [64, 128, 256, 488, 1024])
