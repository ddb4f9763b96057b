"""The oracle's float32 batch_core_blas restatement (oracle/sgns_oracle.c, the CPU
baseline's core; reference kernel_batched.py:92-144).

The reference pins its BLAS backend against the naive one by tolerance
(tests/test_kernel_batched.py:133-140, rtol 2e-5) because BLAS summation order is
unspecified; the same bars are applied here, plus a float64 re-derivation at d = 300.
"""
import numpy as np
import pytest

from oracle import oracle as O
from paper_1604_04661_b200.model import SIGMOID_TABLE_F32


def test_blas_agrees_with_naive_small():
    """The reference's own naive-vs-blas case shape: V=12, D=9, inputs [1,2,3,1], outputs
    [0,5,6,7], alpha 0.05, rtol 2e-5."""
    rng = np.random.default_rng(14)
    a = rng.uniform(-0.5, 0.5, size=(12, 9)).astype(np.float32)
    c = rng.uniform(-0.5, 0.5, size=(12, 9)).astype(np.float32)
    a1, c1, a2, c2 = a.copy(), c.copy(), a.copy(), c.copy()
    ins, outs = np.array([1, 2, 3, 1], np.int32), np.array([0, 5, 6, 7], np.int32)
    O.process_batch(a1, c1, ins, outs, 0.05, SIGMOID_TABLE_F32, "naive")
    O.process_batch(a2, c2, ins, outs, 0.05, SIGMOID_TABLE_F32, "blas")
    np.testing.assert_allclose(a2, a1, rtol=2e-5)
    np.testing.assert_allclose(c2, c1, rtol=2e-5)


@pytest.mark.parametrize("D,m,k1", [(300, 10, 6), (100, 7, 6), (300, 3, 16), (37, 10, 4)])
def test_blas_matches_float64_derivation(D, m, k1):
    """scores = A C^T, g = alpha (label - table(score)), C += g^T A, A += g C (float64
    re-derivation); windows whose float64 score sits within 1e-5 of a sigma-bin edge are
    skipped (either side of the edge is a valid float32 result)."""
    rng = np.random.default_rng(D + m + k1)
    V = 64
    for _ in range(20):
        a = (rng.normal(size=(V, D)) * D ** -0.25).astype(np.float32)
        c = (rng.normal(size=(V, D)) * D ** -0.25).astype(np.float32)
        ins = rng.integers(0, V, m).astype(np.int32)
        outs = rng.choice(V, k1, replace=False).astype(np.int32)
        A, Cm = a[ins].astype(np.float64), c[outs].astype(np.float64)
        s = A @ Cm.T
        v = (s + 6.0) * (1000.0 / 12.0)
        if np.any(np.abs(v - np.rint(v)) < 1e-3):
            continue
        idx = np.clip(np.floor(v).astype(np.int64), 0, 999)
        g = 0.025 * ((np.arange(k1) == 0)[None, :] - SIGMOID_TABLE_F32[idx].astype(np.float64))
        ea, ec = a.astype(np.float64), c.astype(np.float64)
        np.add.at(ec, outs, g.T @ A)
        np.add.at(ea, ins, g @ Cm)
        got_a, got_c = a.copy(), c.copy()
        O.process_batch(got_a, got_c, ins, outs, 0.025, SIGMOID_TABLE_F32, "blas")
        np.testing.assert_allclose(got_a, ea, rtol=1e-5, atol=1e-6)
        np.testing.assert_allclose(got_c, ec, rtol=1e-5, atol=1e-6)


def test_blas_drive_trains_like_naive():
    """The fused CPU driver with the blas core (the bench's CPU baseline) reaches the naive
    core's loss on the same stream (same draws; only the GEMM rounding differs)."""
    from paper_1604_04661_b200.corpus import default_table_length, keep_probabilities
    from paper_1604_04661_b200.synthetic import make_planted_corpus
    syn = make_planted_corpus(60_000, 2_000, zipf_s=1.0, min_count=1, seed=3)
    e, counts = syn.encoded, syn.vocab.counts
    V, D = len(counts), 32
    keep = keep_probabilities(counts, int(counts.sum()), 1e-3)
    L = default_table_length(V)
    slots = np.repeat(np.arange(V, dtype=np.int32), np.diff(O.neg_boundaries(counts, 0.75, L), prepend=0))
    losses = {}
    for mm in ("naive", "blas"):
        m_in = O.init_model(V, D, 1).astype(np.float32)
        m_out = np.zeros((V, D), np.float32)
        run = O.OracleRun(e.ids, e.offsets, m_in, m_out, keep_probs=keep, window=5, negatives=5,
                          batch_cap=16, dynamic=True, seed=1, alpha0=0.025, floor_frac=1e-4,
                          total_x_epochs=float(e.n_tokens) * 2, epochs=2, loss_every=1, n_workers=1,
                          slots=slots, sig_table=SIGMOID_TABLE_F32, matmul=mm)
        while not run.done:
            run.advance(1 << 40, 1)
        losses[mm] = run.loss.sum(axis=0) / run.cells.sum(axis=0)
    np.testing.assert_allclose(losses["blas"], losses["naive"], rtol=2e-3)
