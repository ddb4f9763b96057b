"""Edge cases of the device path: empty and ragged window batches, the
extremes of K (1 and 31 negatives) and of the row width (d = 4 ... 1024 float32, 512
float64), degenerate sentences (empty, one token, the 1,000-token maximum) and a sentence
beyond the kernel envelope.  Tolerances as in test_gpu_parity.py."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from test_gpu_parity import _oracle_philox, _random_windows, _run_driver, near_bin_edge  # noqa: E402


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("needs CUDA")


def _models(V, D, npdt, seed):
    import paper_1604_04661_b200 as P
    rng = np.random.default_rng(seed)
    return P.EmbeddingModel((rng.normal(size=(V, D)) * D ** -0.25).astype(npdt),
                            (rng.normal(size=(V, D)) * D ** -0.25).astype(npdt))


def _apply_snapshot(base, wins, alphas):
    import paper_1604_04661_b200 as P
    from paper_1604_04661_b200.kernel_batched import DeviceWindowBatch, WindowBatch
    from paper_1604_04661_b200.model import DeviceModel
    wb = WindowBatch.from_minibatches([P.Minibatch(a, b) for a, b in wins])
    src = DeviceModel.from_host(base)
    dst = src.clone()
    P.update_windows(dst, DeviceWindowBatch(wb), torch.from_numpy(alphas), src=src)
    return dst.to_host()


def _oracle_snapshot(base, wins, alphas, npdt):
    from oracle import oracle as O
    from paper_1604_04661_b200.model import SIGMOID_TABLE_F32, SIGMOID_TABLE_F64
    tab = SIGMOID_TABLE_F64 if npdt == np.float64 else SIGMOID_TABLE_F32
    acc_in = base.input_vectors.astype(np.float64).copy()
    acc_out = base.output_vectors.astype(np.float64).copy()
    for (a, b), al in zip(wins, alphas):
        mi, mo = base.input_vectors.copy(), base.output_vectors.copy()
        O.process_batch(mi, mo, a, b, float(npdt(al)), tab)
        acc_in += mi.astype(np.float64) - base.input_vectors
        acc_out += mo.astype(np.float64) - base.output_vectors
    return acc_in, acc_out


def test_empty_window_batch_is_a_noop():
    import paper_1604_04661_b200 as P
    from paper_1604_04661_b200.kernel_batched import DeviceWindowBatch, WindowBatch
    from paper_1604_04661_b200.model import DeviceModel
    base = _models(50, 16, np.float32, 0)
    dm = DeviceModel.from_host(base)
    wb = WindowBatch(np.zeros(1, np.int32), np.zeros(0, np.int32), np.zeros((0, 6), np.int32))
    P.update_windows(dm, DeviceWindowBatch(wb), 0.025)
    got = dm.to_host()
    assert np.array_equal(got.input_vectors, base.input_vectors)
    assert np.array_equal(got.output_vectors, base.output_vectors)


@pytest.mark.parametrize("dtype,k", [("f64", 1), ("f64", 31), ("f32", 1), ("f32", 31)])
def test_ragged_windows_extreme_k(dtype, k):
    """m = 1 ... 16 inputs per window, K = 1 (k1 = 2) and K = 31 (k1 = 32, the envelope),
    Zipf-conflicting rows, snapshot mode == snapshot + sum of per-window oracle deltas."""
    npdt = np.float64 if dtype == "f64" else np.float32
    rng = np.random.default_rng(k)
    V, D = 300, 96
    base = _models(V, D, npdt, k)
    wins = _random_windows(rng, V, 160, 16, k)
    wins = [(np.resize(a, 1 + i % 16).astype(np.int32), b) for i, (a, b) in enumerate(wins)]
    alphas = rng.uniform(0.001, 0.03, size=len(wins))
    got = _apply_snapshot(base, wins, alphas)
    acc_in, acc_out = _oracle_snapshot(base, wins, alphas, npdt)
    if dtype == "f64":
        np.testing.assert_allclose(got.input_vectors, acc_in, rtol=1e-10, atol=1e-13)
        np.testing.assert_allclose(got.output_vectors, acc_out, rtol=1e-10, atol=1e-13)
    else:
        from oracle import pin
        from paper_1604_04661_b200.model import SIGMOID_TABLE_F32
        _, mags, allows, _ = pin.snapshot_expectation(base.input_vectors, base.output_vectors, wins,
                                                  alphas, SIGMOID_TABLE_F32, check_edges=True)
        for got_m, acc, mag, allow in zip((got.input_vectors, got.output_vectors), (acc_in, acc_out),
                                         mags, allows):
            worst = pin.snapshot_budget(got_m, acc, mag, allow)
            assert worst <= 1.0, f"tolerance budget used {worst:.3f} (1e-5 |summed| + 1e-7)"


@pytest.mark.parametrize("dtype,D", [("f32", 4), ("f32", 512), ("f32", 516), ("f32", 1024),
                                     ("f64", 2), ("f64", 512)])
def test_row_width_envelope(dtype, D):
    """Smallest and largest rows of each kernel variant (float2 fast path up to 512,
    generic path above; float64 up to 512): disjoint windows == sequential oracle."""
    from oracle import oracle as O
    from paper_1604_04661_b200.model import SIGMOID_TABLE_F32, SIGMOID_TABLE_F64
    npdt = np.float64 if dtype == "f64" else np.float32
    rng = np.random.default_rng(D)
    V, k = 3000, 5
    base = _models(V, D, npdt, D)
    wins = _random_windows(rng, V, 120, 10, k, disjoint=True)
    alphas = np.full(len(wins), 0.025)
    got = _apply_snapshot(base, wins, alphas)
    ref_in, ref_out = base.input_vectors.copy(), base.output_vectors.copy()
    tab = SIGMOID_TABLE_F64 if dtype == "f64" else SIGMOID_TABLE_F32
    flips = 0
    for a, b in wins:
        O.process_batch(ref_in, ref_out, a, b, 0.025, tab)
        s = base.input_vectors[a].astype(np.float64) @ base.output_vectors[b].astype(np.float64).T
        flips += int(near_bin_edge(s).any())
    if dtype == "f64":
        np.testing.assert_allclose(got.input_vectors, ref_in, rtol=1e-12, atol=1e-15)
        np.testing.assert_allclose(got.output_vectors, ref_out, rtol=1e-12, atol=1e-15)
    else:
        bad_in = np.abs(got.input_vectors.astype(np.float64) - ref_in) > 1e-5 * np.abs(ref_in) + 1e-7
        bad_out = np.abs(got.output_vectors.astype(np.float64) - ref_out) > 1e-5 * np.abs(ref_out) + 1e-7
        assert int(bad_in.any(axis=1).sum() + bad_out.any(axis=1).sum()) <= flips * 16


def test_degenerate_sentences_window_stream():
    """Empty sentences, one-token sentences (no context: read, maybe kept, never a window)
    and a 1,000-token sentence (the reference's max_sentence): the production driver's
    windows equal the oracle's, and every token is read exactly once."""
    rng = np.random.default_rng(4)
    V = 60
    lens = [0, 1, 0, 2, 1000, 1, 0, 5, 1, 1000, 0, 3]
    ids = rng.integers(0, V, size=sum(lens)).astype(np.int32)
    ids[:V] = np.arange(V)  # every id occurs
    off = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    counts = np.bincount(ids, minlength=V).astype(np.int64)
    cap = len(ids) * 2 + 10
    for workers in (1, 7):
        run, sampler = _run_driver(ids, off, counts, window=5, k=5, cap=16, dynamic=True, subsample=1e-2,
                                   seed=3, stream_base=0, table_len=None, rng="philox", workers=workers,
                                   epochs=2, trace_cap=cap, schedule="dynamic")
        assert run.dynamic
        got, got_alpha = run.trace_records()
        orc = _oracle_philox(ids, off, counts, sampler.host_alias, W=1, epochs=2, update=False,
                             trace_cap=cap, cap=16, sub=1e-2, seed=3)
        exp, exp_alpha = orc.worker_trace(0)
        key = lambda a, al: np.lexsort(np.column_stack([a, al.view(np.int64)]).T[::-1])
        gi, ei = key(got, got_alpha), key(exp, exp_alpha)
        assert got.shape == exp.shape and len(exp) > 100
        assert np.array_equal(got[gi], exp[ei])
        assert np.array_equal(got_alpha[gi], exp_alpha[ei])
        assert run.words_read == 2 * len(ids)
        assert run.words_trained == orc.workers[0].words_trained
        # no window comes from a sentence shorter than 2 tokens
        short = {s for s, n in enumerate(lens) if n < 2}
        assert not (set(got[:, 2].tolist()) & short)


def test_sentence_beyond_kernel_envelope_is_refused():
    """A sentence longer than the kernel's 1,024-token staging buffer is refused with an
    error, never silently skipped or truncated."""
    V = 40
    ids = (np.arange(1100) % V).astype(np.int32)
    off = np.array([0, 50, 1100], dtype=np.int64)  # sentence 1 holds 1,050 tokens
    counts = np.bincount(ids, minlength=V).astype(np.int64)
    with pytest.raises((RuntimeError, ValueError)):
        _run_driver(ids, off, counts, window=5, k=5, cap=16, dynamic=True, subsample=0.0, seed=1,
                    stream_base=0, table_len=None, rng="philox", workers=4, epochs=1, trace_cap=0,
                    schedule="dynamic")
