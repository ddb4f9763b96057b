"""Window-stream replay checks for the device drivers (TEST INFRASTRUCTURE ONLY).

Used by tests/test_gpu_fast_pin.py and __graft_entry__.smoke() to pin the timed
production kernel (drive_fast_kernel) against the oracle's process_batch, which
restates batch_core_naive (sgns/kernel_batched.py:147-211) and is pinned bit for bit
to the reference's own outputs (tests/test_oracle_golden.py).  The package never
imports this module.
"""

from __future__ import annotations

import numpy as np

from . import oracle as O

# |gpu - oracle| <= RTOL |oracle| + ATOL  (the reference's float32 acceptance metric,
# tests/test_acceptance.py:199-209)
RTOL, ATOL = 1e-5, 1e-7
# A score s can land in the neighbouring sigma bin under another summation order only if
# it lies within the two orders' rounding distance of a bin edge.
# That distance is bounded by a few float32 ulps of the partial sums, i.e. by a small
# multiple of eps32 * sum_j |a_j c_j| (plus the ulp-level drift of the rows themselves in a
# sequential replay).  EDGE_ABS + EDGE_REL * sum_j |a_j c_j| is ~10x the observed distance.
EDGE_ABS, EDGE_REL = 1e-6, 5e-7


def near_edge(scores, l1=None) -> np.ndarray:
    """True for scores within the flip distance of a real bin edge: v = (s + 6) * 1000/12
    at an integer 1..999 (v < 1 and v >= 999 are clamped into bins 0 / 999, so -6 and
    +6 are not edges).  l1: sum_j |a_j c_j| per score (default: |s|)."""
    s = np.asarray(scores, dtype=np.float64)
    l1 = np.abs(s) if l1 is None else np.asarray(l1, dtype=np.float64)
    v = (s + 6.0) * (1000.0 / 12.0)
    e = np.clip(np.round(v), 1.0, 999.0)
    dist = np.abs(v - e) * (12.0 / 1000.0)
    return dist < EDGE_ABS + EDGE_REL * l1


def window_scores(m_in, m_out, ins, outs):
    """float64 scores S = A C^T of one window and the per-cell sums of |a_j c_j|."""
    a = m_in[ins].astype(np.float64)
    c = m_out[outs].astype(np.float64)
    return a @ c.T, np.abs(a) @ np.abs(c).T


def softplus(x):
    """sgns/kernel_scalar.py:38-51 (float64)."""
    x = np.asarray(x, dtype=np.float64)
    return np.maximum(x, 0.0) + np.log1p(np.exp(-np.abs(x)))


def tiny_corpus(rng, V: int, n_sent: int, lo: int, hi: int):
    """Zipf(1)-weighted ids over a tiny vocabulary: consecutive windows share rows."""
    p = 1.0 / np.arange(1, V + 1)
    p /= p.sum()
    lens = rng.integers(lo, hi + 1, size=n_sent)
    ids = rng.choice(V, size=int(lens.sum()), p=p).astype(np.int32)
    counts = np.bincount(ids, minlength=V).astype(np.int64)
    counts[counts == 0] = 1
    off = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    return ids, off, counts


def budget_used(got: np.ndarray, exp: np.ndarray) -> float:
    g = got.astype(np.float64)
    e = exp.astype(np.float64)
    r = np.abs(g - e) / (RTOL * np.abs(e) + ATOL)
    return float(r.max()) if r.size else 0.0


def replay_sentences(run, dm, n_sentences: int, cap: int, k1: int, sig_table) -> dict:
    """Advance a one-worker dynamic-schedule DeviceRun (trace on, loss_every = 1) one
    sentence at a time; replay each sentence's traced windows with the oracle from the
    GPU state before it and compare the GPU state after it.  Returns the tallies."""
    out = dict(compared=0, flagged=0, windows=0, shared_next=0, worst=0.0, loss_worst=0.0)
    n_seen = 0
    loss_prev = 0.0
    for s in range(n_sentences):
        before = dm.to_host()
        run.advance(1)
        recs, alphas = run.trace_records()
        new, new_alpha = recs[n_seen:], alphas[n_seen:]
        n_seen = len(recs)
        if len(new) and not (new[:, 2] == s).all():
            raise AssertionError(f"sentence {s}: trace holds windows of other sentences")
        loss_now = float(run.loss.sum().item())
        gpu_loss, loss_prev = loss_now - loss_prev, loss_now
        mi = before.input_vectors.copy()
        mo = before.output_vectors.copy()
        edge = False
        exp_loss = 0.0
        prev_out = None
        for rec, al in zip(new, new_alpha):
            m = int(rec[1])
            ins = rec[4:4 + m]
            outs = rec[4 + cap:4 + cap + k1]
            if outs[0] != rec[0] or (outs[1:] == outs[0]).any():
                raise AssertionError(f"sentence {s}: bad output ids {outs}")
            sc, l1 = window_scores(mi, mo, ins, outs)
            edge |= bool(near_edge(sc, l1).any())
            exp_loss += float(softplus(-sc[:, 0]).sum() + softplus(sc[:, 1:]).sum())
            O.process_batch(mi, mo, ins, outs, float(np.float32(al)), sig_table, matmul="naive")
            if prev_out is not None and np.intersect1d(prev_out, outs).size:
                out["shared_next"] += 1
            prev_out = outs
            out["windows"] += 1
        if edge:  # a legal bin flip changes the windows after it: model and loss both skipped
            out["flagged"] += 1
            continue
        if len(new):
            out["loss_worst"] = max(out["loss_worst"], abs(gpu_loss - exp_loss) / (1e-5 * abs(exp_loss) + 1e-9))
        after = dm.to_host()
        out["worst"] = max(out["worst"], budget_used(after.input_vectors, mi),
                           budget_used(after.output_vectors, mo))
        out["compared"] += 1
    return out


def snapshot_expectation(m_in, m_out, wins, alphas, sig_table, check_edges: bool):
    """Snapshot mode (every window reads the same model, deltas accumulate): returns the
    float64 sums snapshot + sum_w delta_w, the magnitudes |snapshot| + sum_w |delta_w|
    that bound float32 summation in any order, and the bin-flip allowances: for every
    cell (i, k) whose score sits at a sigma-bin edge, the other bin moves err by the
    table step dsig there, i.e. row in_i by alpha dsig |c_k| and row out_k by alpha dsig
    |a_i| ("recompute each mismatching cell with the other side's bin")."""
    npdt = m_in.dtype
    acc_in, acc_out = m_in.astype(np.float64), m_out.astype(np.float64)
    mag_in, mag_out = np.abs(acc_in), np.abs(acc_out)
    allow_in = np.zeros_like(acc_in)
    allow_out = np.zeros_like(acc_out)
    tab = np.asarray(sig_table, dtype=np.float64)
    flagged = 0
    for (a, b), al in zip(wins, alphas):
        mi, mo = m_in.copy(), m_out.copy()
        al = npdt.type(al)
        O.process_batch(mi, mo, a, b, float(al), sig_table)
        d_in = mi.astype(np.float64) - m_in
        d_out = mo.astype(np.float64) - m_out
        acc_in += d_in
        acc_out += d_out
        mag_in += np.abs(d_in)
        mag_out += np.abs(d_out)
        if check_edges:
            sc, l1 = window_scores(m_in, m_out, a, b)
            near = near_edge(sc, l1)
            for i, k in zip(*np.nonzero(near)):
                e = int(np.clip(np.round((sc[i, k] + 6.0) * (1000.0 / 12.0)), 1, 999))
                step = abs(tab[e] - tab[e - 1]) * float(al) * 1.01
                allow_in[a[i]] += step * np.abs(m_out[b[k]].astype(np.float64))
                allow_out[b[k]] += step * np.abs(m_in[a[i]].astype(np.float64))
                flagged += 1
    return (acc_in, acc_out), (mag_in, mag_out), (allow_in, allow_out), flagged


def snapshot_budget(got, acc, mag, allow) -> float:
    """Worst (|got - acc| - allow) / (RTOL * mag + ATOL): <= 1 passes."""
    r = (np.abs(got.astype(np.float64) - acc) - allow) / (RTOL * mag + ATOL)
    return float(r.max()) if r.size else 0.0
