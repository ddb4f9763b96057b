"""Test helpers (imported as a plain module: tests/ is on sys.path under pytest)."""

import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def load_golden(name: str):
    return np.load(os.path.join(GOLDEN, f"{name}.npz"), allow_pickle=False)


def kernel_case(g, i):
    """(V, D, base f64 model pair, in_ids, out_ids, alpha) of golden kernel case i."""
    m_in = g[f"c{i}_min"]
    m_out = g[f"c{i}_mout"]
    return (m_in, m_out, g[f"c{i}_in_ids"], g[f"c{i}_out_ids"], float(g[f"c{i}_alpha"][0]),
            g[f"c{i}_rows_in"], g[f"c{i}_rows_out"])


TRAIN_CASES = {
    # mirrors tests/golden/make_golden.py TRAIN_CASES (base + overrides)
    "f64_naive": dict(float64=True),
    "f32_naive": dict(float64=False, matmul="naive"),
    "f32_blas": dict(float64=False),
    "f64_cap1_k1": dict(float64=True, batch_cap=1, negatives=1),
    "f64_w10_cap4": dict(float64=True, window=10, batch_cap=4, negatives=3),
    "f64_static_nosub": dict(float64=True, dynamic_window=False, subsample=0.0),
    "f32_k15_loss1": dict(float64=False, negatives=15, loss_sample_every=1, matmul="naive"),
    "f64_loss7": dict(float64=True, loss_sample_every=7, epochs=3),
}
TRAIN_BASE = dict(dim=16, window=5, negatives=5, subsample=1e-3, min_count=1, alpha0=0.025,
                  epochs=2, threads=1, batch_cap=16, kernel="batched", seed=3,
                  dynamic_window=True, float64=False, loss_sample_every=100)


def train_config(name):
    cfg = dict(TRAIN_BASE)
    cfg.update(TRAIN_CASES[name])
    return cfg


TRACE_CASES = [
    # name, n_tokens, V, window, K, cap, dynamic, subsample, seed, stream, table_len
    ("t0", 4000, 60, 5, 5, 16, True, 1e-2, 1, 0, None),
    ("t1", 4000, 60, 10, 4, 3, True, 1e-2, 7, 2, None),
    ("t2", 3000, 40, 2, 2, 4, False, 0.0, 3, 5, 997),
    ("t3", 6000, 200, 5, 15, 16, True, 1e-3, 11, 0x1017, None),
]


def trace_to_records(g, name, cap, k1):
    """Golden pipeline trace -> the oracle/device record layout [target, m, sent, epoch, in.., out..]."""
    tgt = g[f"{name}_target"]
    off = g[f"{name}_in_off"]
    ins = g[f"{name}_in_ids"]
    outs = g[f"{name}_out_ids"]
    sent = g[f"{name}_sentence"]
    recs = np.full((len(tgt), 4 + cap + k1), -1, dtype=np.int32)
    for r in range(len(tgt)):
        m = off[r + 1] - off[r]
        recs[r, 0] = tgt[r]
        recs[r, 1] = m
        recs[r, 2] = sent[r]
        recs[r, 3] = 0
        recs[r, 4:4 + m] = ins[off[r]:off[r + 1]]
        recs[r, 4 + cap:] = outs[r]
    return recs
