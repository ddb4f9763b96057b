"""GPU parity: the CUDA path (through the C ABI) against the oracle and the
reference-generated golden fixtures.  Tolerances are written in each test:
  float64: rtol 1e-12 per update (tree vs sequential summation order only),
  float32: |a - b| <= 1e-5 |a| + 1e-7 (tests/test_acceptance.py:199-209),
  integers (windows, chunks, negatives, counters): bit-exact.
"""

import numpy as np
import pytest

from helpers import TRACE_CASES, kernel_case, load_golden, trace_to_records, train_config

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("needs CUDA")
    torch.cuda.set_device(0)


def _pkg():
    import paper_1604_04661_b200 as P
    return P


def _oracle():
    from oracle import oracle as O
    return O


def f32_close(a, b, rtol=1e-5, atol=1e-7):
    ratio = np.abs(a.astype(np.float64) - b.astype(np.float64)) / (rtol * np.abs(b.astype(np.float64)) + atol)
    return float(ratio.max()) if ratio.size else 0.0


def near_bin_edge(scores, tol=2e-5):
    v = (np.asarray(scores, dtype=np.float64) + 6.0) * (1000.0 / 12.0)
    return np.abs(v - np.round(v)) < tol * 1000.0 / 12.0 * np.maximum(1.0, np.abs(scores))


def test_graft_smoke():
    import __graft_entry__ as g
    g.smoke()


def test_library_is_the_one_loaded():
    from paper_1604_04661_b200 import _lib
    L = _lib.lib()
    maps = open("/proc/self/maps").read()
    assert _lib.LIB_PATH in maps
    assert L.sgns_abi_version() == 2


@pytest.mark.parametrize("dtype", ["f64", "f32"])
def test_process_batch_golden(dtype):
    """P1: one minibatch vs the reference's own process_batch outputs."""
    P = _pkg()
    g = load_golden("kernel")
    npdt = np.float64 if dtype == "f64" else np.float32
    worst = 0.0
    for i in range(int(g["n_cases"][0])):
        m_in, m_out, ins, outs, alpha, r_in, r_out = kernel_case(g, i)
        model = P.EmbeddingModel(m_in.astype(npdt), m_out.astype(npdt))
        before = model.copy()
        P.process_batch(model, P.Minibatch(ins, outs), alpha)
        # locality: untouched rows bit-identical
        mask_in = np.ones(len(m_in), bool)
        mask_in[r_in] = False
        mask_out = np.ones(len(m_out), bool)
        mask_out[r_out] = False
        assert np.array_equal(model.input_vectors[mask_in], before.input_vectors[mask_in])
        assert np.array_equal(model.output_vectors[mask_out], before.output_vectors[mask_out])
        if alpha == 0.0:
            assert np.array_equal(model.input_vectors, before.input_vectors)
            assert np.array_equal(model.output_vectors, before.output_vectors)
        if dtype == "f64":
            np.testing.assert_allclose(model.input_vectors[r_in], g[f"c{i}_f64_naive_min"], rtol=1e-12, atol=1e-15)
            np.testing.assert_allclose(model.output_vectors[r_out], g[f"c{i}_f64_naive_mout"], rtol=1e-12, atol=1e-15)
        else:
            scores = before.input_vectors[ins].astype(np.float64) @ before.output_vectors[outs].astype(np.float64).T
            if near_bin_edge(scores).any():
                continue  # a sigma-table bin flip between summation orders is legal
            for be in ("naive", "blas"):
                worst = max(worst, f32_close(model.input_vectors[r_in], g[f"c{i}_f32_{be}_min"]))
                worst = max(worst, f32_close(model.output_vectors[r_out], g[f"c{i}_f32_{be}_mout"]))
    assert worst <= 1.0, f"float32 tolerance budget used {worst:.2f}"


@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_process_batch_host_row_granular(dtype, monkeypatch):
    """Host models move only the window's distinct rows (kernel_batched.py:214-260 gathers
    and scatters just those): repeated inputs, an input equal to an output id, V = 200k;
    the result equals the oracle's in-place update and the device model allocated is
    (distinct rows) x D, not V x D."""
    P, O = _pkg(), _oracle()
    from paper_1604_04661_b200 import model as M
    from paper_1604_04661_b200.model import SIGMOID_TABLE_F32, SIGMOID_TABLE_F64
    rng = np.random.default_rng(4)  # no float32 score within the bin-flip distance of an edge
    V, D = 200_000, 96
    a = (rng.normal(size=(V, D)) * 0.1).astype(dtype)
    c = (rng.normal(size=(V, D)) * 0.1).astype(dtype)
    ins = np.array([7, 199_999, 7, 42, 5, 7], np.int32)
    outs = np.array([42, 0, 199_998, 5, 12], np.int32)
    sizes = []
    orig = M.DeviceModel.empty.__func__

    def spy(cls, vocab_size, dim, dtype=np.float32, device="cuda"):
        sizes.append(vocab_size)
        return orig(cls, vocab_size, dim, dtype, device)
    monkeypatch.setattr(M.DeviceModel, "empty", classmethod(spy))
    model = P.EmbeddingModel(a.copy(), c.copy())
    P.process_batch(model, P.Minibatch(ins, outs), 0.05)
    assert sizes and max(sizes) <= len(ins) + len(outs), sizes
    ra, rc = a.copy(), c.copy()
    tab = SIGMOID_TABLE_F64 if dtype == np.float64 else SIGMOID_TABLE_F32
    O.process_batch(ra, rc, ins, outs, 0.05, tab)
    if dtype == np.float64:
        np.testing.assert_allclose(model.input_vectors, ra, rtol=1e-12, atol=1e-15)
        np.testing.assert_allclose(model.output_vectors, rc, rtol=1e-12, atol=1e-15)
    else:
        assert not near_bin_edge(a[ins].astype(np.float64) @ c[outs].astype(np.float64).T).any()
        assert f32_close(model.input_vectors, ra) <= 1.0
        assert f32_close(model.output_vectors, rc) <= 1.0
    touched_in = np.zeros(V, bool)
    touched_in[ins] = True
    touched_out = np.zeros(V, bool)
    touched_out[outs] = True
    assert np.array_equal(model.input_vectors[~touched_in], a[~touched_in])
    assert np.array_equal(model.output_vectors[~touched_out], c[~touched_out])


def test_process_batch_validation():
    P = _pkg()
    m = P.EmbeddingModel(np.zeros((5, 4), np.float32), np.zeros((5, 4), np.float32))
    with pytest.raises(ValueError):
        P.process_batch(m, P.Minibatch([1], [0, 2]), -0.1)
    with pytest.raises(ValueError):
        P.process_batch(m, P.Minibatch([1], [0, 2]), 0.1, matmul="magic")
    P.process_batch(m, P.Minibatch([1], [0, 2]), 0.1, matmul="blas")  # reference names accepted
    P.process_batch(m, P.Minibatch([1], [0, 2]), 0.1, matmul="naive")
    with pytest.raises(ValueError):
        P.Minibatch([1], [3, 3])
    with pytest.raises(ValueError):
        P.process_batch(m, P.Minibatch([7], [0, 2]), 0.1)


def test_init_model_bitwise():
    P = _pkg()
    g = load_golden("init")
    for key in g.files:
        if not key.startswith("in64_"):
            continue
        _, V, D, seed = key.split("_")
        m64 = P.init_model(int(V), int(D), int(seed), dtype=np.float64)
        m32 = P.init_model(int(V), int(D), int(seed), dtype=np.float32)
        assert np.array_equal(m64.input_vectors, g[key])
        assert np.array_equal(m32.input_vectors, g["in32_" + key[5:]])
        assert not m32.output_vectors.any()


def _random_windows(rng, V, n, m_max, k, disjoint=False, m_fixed=None):
    wins = []
    pool = rng.permutation(V)
    used = 0
    for _ in range(n):
        m = int(rng.integers(1, m_max + 1)) if m_fixed is None else m_fixed
        if disjoint:
            ids = pool[used:used + m + k + 1]
            used += m + k + 1
            ins, outs = ids[:m], ids[m:]
        else:
            zipf = np.minimum(rng.zipf(1.3, size=m + k + 1) - 1, V - 1)
            ins, outs = zipf[:m], zipf[m:]
            while (outs[1:] == outs[0]).any():
                outs[1:] = np.where(outs[1:] == outs[0], rng.integers(0, V, k), outs[1:])
        wins.append((np.asarray(ins, np.int32), np.asarray(outs, np.int32)))
    return wins


@pytest.mark.parametrize("dtype,D,k", [("f64", 300, 5), ("f32", 300, 5), ("f32", 100, 5),
                                       ("f32", 200, 10), ("f32", 300, 15), ("f32", 512, 15),
                                       ("f32", 64, 8), ("f32", 40, 12), ("f32", 300, 16),
                                       ("f64", 24, 3)])
def test_disjoint_windows_equal_sequential(dtype, D, k):
    """P2: a batch of row-disjoint windows == the sequential oracle application."""
    _p2_disjoint(dtype, D, k)


@pytest.mark.parametrize("dtype,D,k,ld", [("f32", 300, 5, 300), ("f32", 300, 5, 304), ("f32", 300, 15, 300),
                                          ("f32", 100, 12, 100), ("f32", 200, 10, 256), ("f64", 30, 3, 30),
                                          ("f64", 300, 5, 302)])
def test_disjoint_windows_any_row_stride(dtype, D, k, ld):
    """P2 on models whose row stride is not the package's own (model.py padded_ld): the C
    ABI takes any stride that is a multiple of 16 bytes; only the dim data columns are
    touched, staged rows are packed at the data width."""
    _p2_disjoint(dtype, D, k, ld)


def _p2_disjoint(dtype, D, k, ld=None):
    P, O = _pkg(), _oracle()
    from paper_1604_04661_b200.kernel_batched import DeviceWindowBatch, WindowBatch
    from paper_1604_04661_b200.model import DeviceModel, SIGMOID_TABLE_F32, SIGMOID_TABLE_F64
    rng = np.random.default_rng(D + k)
    npdt = np.float64 if dtype == "f64" else np.float32
    V = 4000
    scale = D ** -0.25
    base = P.EmbeddingModel((rng.normal(size=(V, D)) * scale).astype(npdt),
                            (rng.normal(size=(V, D)) * scale).astype(npdt))
    wins = _random_windows(rng, V, 150, 10, k, disjoint=True)
    alpha = 0.025
    wb = WindowBatch.from_minibatches([P.Minibatch(a, b) for a, b in wins])
    if ld is None:
        dm = DeviceModel.from_host(base)
    else:
        st = torch.full((2, V, ld), 7.0, dtype=torch.float64 if dtype == "f64" else torch.float32, device="cuda")
        st[0, :, :D].copy_(torch.from_numpy(base.input_vectors))
        st[1, :, :D].copy_(torch.from_numpy(base.output_vectors))
        dm = DeviceModel(st[0], st[1], D, st)
    P.update_windows(dm, DeviceWindowBatch(wb), alpha)
    got = dm.to_host()
    if ld is not None and ld > D:  # the pad columns are never written
        assert bool((dm.storage[:, :, D:] == 7.0).all())
    ref_in, ref_out = base.input_vectors.copy(), base.output_vectors.copy()
    tab = SIGMOID_TABLE_F64 if dtype == "f64" else SIGMOID_TABLE_F32
    flips = 0
    for a, b in wins:
        O.process_batch(ref_in, ref_out, a, b, alpha, tab)
        s = base.input_vectors[a].astype(np.float64) @ base.output_vectors[b].astype(np.float64).T
        flips += int(near_bin_edge(s).any())
    if dtype == "f64":
        np.testing.assert_allclose(got.input_vectors, ref_in, rtol=1e-12, atol=1e-15)
        np.testing.assert_allclose(got.output_vectors, ref_out, rtol=1e-12, atol=1e-15)
    else:
        bad_in = np.abs(got.input_vectors.astype(np.float64) - ref_in) > 1e-5 * np.abs(ref_in) + 1e-7
        bad_out = np.abs(got.output_vectors.astype(np.float64) - ref_out) > 1e-5 * np.abs(ref_out) + 1e-7
        bad_rows = int(bad_in.any(axis=1).sum() + bad_out.any(axis=1).sum())
        # only windows with a score on a sigma-bin edge may differ (<= their rows)
        assert bad_rows <= flips * 16, (bad_rows, flips)


@pytest.mark.parametrize("dtype,D,k,body", [("f64", 300, 5, ""), ("f32", 300, 5, ""), ("f32", 100, 12, ""),
                                            ("f32", 64, 7, ""), ("f32", 100, 5, ""), ("f32", 300, 15, ""),
                                            ("f32", 200, 10, ""), ("f32", 300, 9, ""), ("f32", 300, 15, "s"),
                                            ("f32", 100, 12, "g"), ("f32", 300, 10, "s")])
def test_snapshot_conflicting_windows(dtype, D, k, body, monkeypatch):
    """P3: Zipf-conflicting windows in snapshot mode == snapshot + sum of per-window deltas.

    float32 snapshot mode sums the hottest rows per warp before one scatter: rows [0, 8) of
    both matrices in shared memory where it fits (d = 64, 100, 200), row 0 of M_in in
    registers otherwise (d = 300).  8 < K + 1 <= 16 takes the two-register-group body (F2G)
    or the all-staged one (F2S), as the launcher chooses ("") or forced ("g" / "s").
    Zipf(1.3) puts id 0 in ~30% of the slots here."""
    if body:
        monkeypatch.setenv("SGNS_UPDATE_BODY", body)
    _p3_snapshot(dtype, D, k)


@pytest.mark.parametrize("D", [100, 200, 300])
@pytest.mark.parametrize("w", [2, 5, 10])
@pytest.mark.parametrize("k", [5, 10, 15])
def test_snapshot_configs1_grid(D, w, k):
    """P3 on every shape of BASELINE.json configs[1] (d x w x K, full windows m = 2w as the
    microbench runs them: `bench.py --config micro --micro-grid`), Zipf-conflicting rows."""
    _p3_snapshot("f32", D, k, m_fixed=2 * w, n_win=300)


@pytest.mark.parametrize("D,k,m", [(100, 15, 20), (128, 12, 7), (36, 9, 20)])
def test_snapshot_wide_body_forced(D, k, m, monkeypatch):
    """The d <= 128 single-group body (window_update_f2w) on shapes the launcher would give
    to the two-group body (K + 1 > 12 with more than 12 inputs) or to other row widths."""
    monkeypatch.setenv("SGNS_UPDATE_BODY", "w")
    _p3_snapshot("f32", D, k, m_fixed=m, n_win=300)


@pytest.mark.parametrize("D,k,m", [(100, 5, 20), (300, 5, 13), (64, 12, 15), (300, 15, 20), (200, 10, 3)])
def test_snapshot_input_chunks_forced(D, k, m, monkeypatch):
    """Snapshot-mode launches may stage a long window's inputs in two chunks against the same
    outputs (launch_update_t: when 20 staged rows cost resident warps); forced here on shapes
    the launcher would not split, with odd and short windows."""
    monkeypatch.setenv("SGNS_UPDATE_SPLIT", "1")
    _p3_snapshot("f32", D, k, m_fixed=m, n_win=300)


def _p3_snapshot(dtype, D, k, m_fixed=None, n_win=400):
    P, O = _pkg(), _oracle()
    from paper_1604_04661_b200.kernel_batched import DeviceWindowBatch, WindowBatch
    from paper_1604_04661_b200.model import DeviceModel, SIGMOID_TABLE_F32, SIGMOID_TABLE_F64
    rng = np.random.default_rng(7 + D + k + (0 if m_fixed is None else 1000 * m_fixed))
    npdt = np.float64 if dtype == "f64" else np.float32
    V = 500
    base = P.EmbeddingModel((rng.normal(size=(V, D)) * D ** -0.25).astype(npdt),
                            (rng.normal(size=(V, D)) * D ** -0.25).astype(npdt))
    wins = _random_windows(rng, V, n_win, 10, k, m_fixed=m_fixed)
    wb = WindowBatch.from_minibatches([P.Minibatch(a, b) for a, b in wins])
    alphas = rng.uniform(0.001, 0.03, size=len(wins))
    src = DeviceModel.from_host(base)
    dst = src.clone()
    P.update_windows(dst, DeviceWindowBatch(wb), torch.from_numpy(alphas), src=src)
    got = dst.to_host()
    tab = SIGMOID_TABLE_F64 if dtype == "f64" else SIGMOID_TABLE_F32
    from oracle import pin
    (acc_in, acc_out), mags, allows, _ = pin.snapshot_expectation(
        base.input_vectors, base.output_vectors, wins, alphas, tab, check_edges=dtype == "f32")
    if dtype == "f64":
        np.testing.assert_allclose(got.input_vectors, acc_in, rtol=1e-10, atol=1e-13)
        np.testing.assert_allclose(got.output_vectors, acc_out, rtol=1e-10, atol=1e-13)
    else:
        # float32 adds arrive in an unspecified order (atomics, per-warp hot-row sums), so the
        # bound is 1e-5 relative to the magnitude summed, |snapshot| + sum_w |delta_w|, plus
        # 1e-7, plus the table step of each cell whose score sits at a sigma-bin edge
        for got_m, acc, mag, allow in zip((got.input_vectors, got.output_vectors), (acc_in, acc_out),
                                         mags, allows):
            worst = pin.snapshot_budget(got_m, acc, mag, allow)
            assert worst <= 1.0, f"tolerance budget used {worst:.3f}"


def _run_driver(ids, off, counts, *, window, k, cap, dynamic, subsample, seed, stream_base,
                table_len, rng, workers=1, dtype=np.float32, dim=4, epochs=1, update=False,
                model=None, trace_cap=None, loss_every=100, refresh=None, alpha0=0.025,
                schedule="static"):
    P = _pkg()
    from paper_1604_04661_b200.corpus import EncodedCorpus, keep_probabilities
    from paper_1604_04661_b200.model import DeviceModel
    from paper_1604_04661_b200.trainer import DeviceCorpus, DeviceRun, DeviceSampler
    enc = EncodedCorpus(ids, off, np.zeros(len(off) - 1, np.int64))
    cfg = P.TrainingConfig(dim=dim, window=window, negatives=k, batch_cap=cap, dynamic_window=dynamic,
                           subsample=subsample, seed=seed, epochs=epochs, rng=rng, workers=workers,
                           float64=dtype == np.float64, table_length=table_len, min_count=1,
                           loss_sample_every=loss_every, alpha_refresh_words=refresh, alpha0=alpha0,
                           schedule=schedule)
    dm = model if model is not None else DeviceModel.empty(len(counts), dim, dtype)
    corpus = DeviceCorpus(enc)
    sampler = DeviceSampler(counts, rng, table_len)
    keep = keep_probabilities(counts, int(counts.sum()), subsample) if subsample > 0 else None
    if trace_cap is None:
        trace_cap = len(ids) * epochs * (-(-2 * window // cap)) + 10
    run = DeviceRun(dm, corpus, sampler, keep, cfg, alpha0, float(off[-1]) * epochs, workers,
                    stream_base=stream_base, trace_cap=trace_cap, update=update)
    run.run_to_completion()
    return run, sampler


@pytest.mark.parametrize("case", TRACE_CASES, ids=[c[0] for c in TRACE_CASES])
def test_driver_windows_bit_exact_vs_reference(case):
    """Subsample -> dynamic window -> chunks -> shared negatives: the device stream is the
    reference's stream (splitmix, slot table), record for record."""
    name, n, V, w, k, cap, dyn, sub, seed, stream, table_len = case
    g = load_golden("traces")
    ids, off, counts = g[f"{name}_ids"], g[f"{name}_offsets"], g[f"{name}_counts"]
    run, _ = _run_driver(ids, off, counts, window=w, k=k, cap=cap, dynamic=dyn, subsample=sub,
                         seed=seed, stream_base=stream, table_len=table_len, rng="splitmix")
    got, _ = run.worker_trace(0)
    expect = trace_to_records(g, name, cap, k + 1)
    assert got.shape == expect.shape
    assert np.array_equal(got, expect)
    assert int(run.state()["rng"][0]) == int(g[f"{name}_final_state"][0])


@pytest.mark.parametrize("rng_mode", ["splitmix", "philox"])
def test_driver_multiworker_trace_vs_oracle(rng_mode):
    """W workers over split_by_tokens ranges, 2 epochs: per-worker records equal the oracle's."""
    O = _oracle()
    from paper_1604_04661_b200.synthetic import make_planted_corpus
    from paper_1604_04661_b200.corpus import default_table_length, keep_probabilities
    syn = make_planted_corpus(20_000, 300, n_clusters=4, cluster_size=5, sentence_len=41, seed=5)
    ids, off, counts = syn.encoded.ids, syn.encoded.offsets, syn.vocab.counts
    W, w, k, cap = 5, 5, 5, 4
    run, sampler = _run_driver(ids, off, counts, window=w, k=k, cap=cap, dynamic=True, subsample=1e-3,
                               seed=9, stream_base=0, table_len=None, rng=rng_mode, workers=W,
                               epochs=2)
    keep = keep_probabilities(counts, int(counts.sum()), 1e-3)
    slots = alias = None
    if rng_mode == "splitmix":
        L = default_table_length(len(counts))
        slots = np.repeat(np.arange(len(counts), dtype=np.int32),
                          np.diff(O.neg_boundaries(counts, 0.75, L), prepend=0))
    else:
        alias = sampler.host_alias
    m = np.zeros((len(counts), 4), np.float32)
    orc = O.OracleRun(ids, off, m, m.copy(), keep_probs=keep, window=w, negatives=k, batch_cap=cap,
                      dynamic=True, seed=9, alpha0=0.025, floor_frac=1e-4,
                      total_x_epochs=float(off[-1]) * 2, epochs=2, loss_every=0, n_workers=W,
                      rng_mode=rng_mode, slots=slots, alias=alias,
                      sig_table=np.zeros(1000, np.float32), trace_cap=len(ids) * 2 * 3 + 10,
                      update=False, refresh_words=10_000 if rng_mode == "splitmix" else 1)
    orc.run_to_completion()
    st = run.state()
    for wk in range(W):
        a, _ = run.worker_trace(wk)
        b, _ = orc.worker_trace(wk)
        assert a.shape == b.shape and np.array_equal(a, b), wk
        assert int(st["words_read"][wk]) == orc.workers[wk].words_read
        assert int(st["words_trained"][wk]) == orc.workers[wk].words_trained
        assert int(st["kernel_counter"][wk]) == orc.workers[wk].kernel_counter


@pytest.mark.parametrize("name", ["f64_naive", "f64_cap1_k1", "f64_w10_cap4", "f64_static_nosub",
                                  "f64_loss7"])
def test_driver_train_f64_matches_reference(name):
    """Fused driver, one worker, float64: the reference's train_encoded model and stats."""
    P = _pkg()
    cfg = train_config(name)
    g = load_golden("train")
    from paper_1604_04661_b200.corpus import EncodedCorpus, Vocabulary
    enc = EncodedCorpus(g["ids"], g["offsets"], g["sentence_bytes"])
    vocab = Vocabulary.from_counts(g["counts"])
    tc = P.TrainingConfig(**{k: v for k, v in cfg.items()}, rng="splitmix")
    model, stats = P.train_encoded(vocab, enc, tc)
    assert [stats.words_processed, stats.words_read] == g[f"{name}_stats"].tolist()
    assert stats.final_alpha == pytest.approx(float(g[f"{name}_final_alpha"][0]), rel=1e-12)
    np.testing.assert_allclose(stats.loss_by_epoch, g[f"{name}_loss"], rtol=1e-9)
    np.testing.assert_allclose(model.input_vectors, g[f"{name}_min"], rtol=1e-8, atol=1e-12)
    np.testing.assert_allclose(model.output_vectors, g[f"{name}_mout"], rtol=1e-8, atol=1e-12)


@pytest.mark.parametrize("name", ["f32_naive", "f32_blas", "f32_k15_loss1"])
def test_driver_train_f32_close_to_reference(name):
    """float32, one worker: identical stream and counters; loss within 0.5%, model close."""
    P = _pkg()
    cfg = train_config(name)
    g = load_golden("train")
    from paper_1604_04661_b200.corpus import EncodedCorpus, Vocabulary
    enc = EncodedCorpus(g["ids"], g["offsets"], g["sentence_bytes"])
    vocab = Vocabulary.from_counts(g["counts"])
    tc = P.TrainingConfig(**{k: v for k, v in cfg.items() if k != "matmul"}, rng="splitmix")
    model, stats = P.train_encoded(vocab, enc, tc)
    assert [stats.words_processed, stats.words_read] == g[f"{name}_stats"].tolist()
    np.testing.assert_allclose(stats.loss_by_epoch, g[f"{name}_loss"], rtol=5e-3)
    err = np.abs(model.input_vectors - g[f"{name}_min"]).max()
    assert err < 5e-3 * np.abs(g[f"{name}_min"]).max()


def _oracle_philox(syn_ids, off, counts, alias, *, W, epochs, update, m_in=None, m_out=None,
                   loss_every=0, trace_cap=0, window=5, k=5, cap=16, sub=1e-3, seed=9):
    O = _oracle()
    from paper_1604_04661_b200.corpus import keep_probabilities
    from paper_1604_04661_b200.model import SIGMOID_TABLE_F32
    keep = keep_probabilities(counts, int(counts.sum()), sub)
    if m_in is None:
        m_in = np.zeros((len(counts), 4), np.float32)
        m_out = m_in.copy()
    run = O.OracleRun(syn_ids, off, m_in, m_out, keep_probs=keep, window=window, negatives=k,
                      batch_cap=cap, dynamic=True, seed=seed, alpha0=0.025, floor_frac=1e-4,
                      total_x_epochs=float(off[-1]) * epochs, epochs=epochs, loss_every=loss_every,
                      n_workers=W, rng_mode="philox", alias=alias, sig_table=SIGMOID_TABLE_F32,
                      trace_cap=trace_cap, update=update, position_mode=True)
    run.run_to_completion()
    return run


@pytest.mark.parametrize("workers", [1, 300])
def test_fast_driver_windows_match_oracle(workers):
    """Dynamic schedule (sgns_fast.cuh): the multiset of (sentence, epoch, target, inputs,
    negatives, alpha) records equals the oracle's for any worker count (position-keyed draws,
    position-based alpha)."""
    from paper_1604_04661_b200.synthetic import make_planted_corpus
    syn = make_planted_corpus(30_000, 400, n_clusters=4, cluster_size=5, sentence_len=37, seed=6)
    ids, off, counts = syn.encoded.ids, syn.encoded.offsets, syn.vocab.counts
    cap = len(ids) * 2 * 2 + 10
    run, sampler = _run_driver(ids, off, counts, window=5, k=5, cap=6, dynamic=True, subsample=1e-3,
                               seed=9, stream_base=0, table_len=None, rng="philox", workers=workers,
                               epochs=2, trace_cap=cap, schedule="dynamic")
    assert run.dynamic
    got, got_alpha = run.trace_records()
    orc = _oracle_philox(ids, off, counts, sampler.host_alias, W=1, epochs=2, update=False,
                         trace_cap=cap, cap=6)
    exp, exp_alpha = orc.worker_trace(0)
    assert got.shape == exp.shape
    key = lambda a, al: np.lexsort(np.column_stack([a, al.view(np.int64)]).T[::-1])
    gi, ei = key(got, got_alpha), key(exp, exp_alpha)
    assert np.array_equal(got[gi], exp[ei])
    assert np.array_equal(got_alpha[gi], exp_alpha[ei])
    assert run.words_read == orc.workers[0].words_read
    assert run.words_trained == orc.workers[0].words_trained


@pytest.mark.parametrize("D,k", [(64, 5), (300, 7), (512, 2), (100, 3), (320, 5), (4, 6),
                                 (200, 4), (300, 6)])
def test_fast_driver_single_worker_trains_like_oracle(D, k):
    """One worker, dynamic schedule: same windows in the same order -> fp32 model within
    accumulated rounding of the oracle's float64-accumulating restatement; loss within 1e-3.
    Covers the fast kernel's variants: exact K1 = 4..8 (k = 3..7), K1 < 4 padded to 6
    (k = 2), whole-slot rows (d = 64, 320, 512) and partial last slots (d = 4, 100, 200,
    300)."""
    P = _pkg()
    from paper_1604_04661_b200.synthetic import make_planted_corpus
    from paper_1604_04661_b200.model import DeviceModel
    O = _oracle()
    syn = make_planted_corpus(30_000, 400, n_clusters=4, cluster_size=5, sentence_len=37, seed=7)
    ids, off, counts = syn.encoded.ids, syn.encoded.offsets, syn.vocab.counts
    V = len(counts)
    base = O.init_model(V, D, 3).astype(np.float32)
    dm = DeviceModel.from_host(P.EmbeddingModel(base.copy(), np.zeros_like(base)))
    run, sampler = _run_driver(ids, off, counts, window=5, k=k, cap=16, dynamic=True, subsample=1e-3,
                               seed=9, stream_base=0, table_len=None, rng="philox", workers=1,
                               epochs=2, update=True, model=dm, dim=D, loss_every=3, trace_cap=0,
                               schedule="dynamic")
    assert run.dynamic
    m_in, m_out = base.copy(), np.zeros_like(base)
    orc = _oracle_philox(ids, off, counts, sampler.host_alias, W=1, epochs=2, update=True,
                         m_in=m_in, m_out=m_out, loss_every=3, k=k)
    got = dm.to_host()
    np.testing.assert_allclose(run.loss_by_epoch(), orc.stats()[2], rtol=1e-3)
    assert np.abs(got.input_vectors - m_in).max() < 1e-3 * np.abs(m_in).max()
    assert np.abs(got.output_vectors - m_out).max() < 1e-3 * np.abs(m_out).max()


def test_streaming_chunks_equal_resident_training():
    """StreamingTrainer.train_chunks (double-buffered, one worker) trains exactly what the
    resident dynamic-schedule run trains on the same corpus: same windows -> same model."""
    P = _pkg()
    from paper_1604_04661_b200.synthetic import make_planted_corpus
    from paper_1604_04661_b200.model import DeviceModel
    from paper_1604_04661_b200.trainer import StreamingTrainer
    syn = make_planted_corpus(40_000, 500, n_clusters=4, cluster_size=5, sentence_len=37, seed=8)
    ids, off, counts = syn.encoded.ids, syn.encoded.offsets, syn.vocab.counts
    V, D = len(counts), 64
    base = np.random.default_rng(1).normal(size=(V, D)).astype(np.float32) * 0.1
    dm1 = DeviceModel.from_host(P.EmbeddingModel(base.copy(), np.zeros_like(base)))
    run, _ = _run_driver(ids, off, counts, window=5, k=5, cap=16, dynamic=True, subsample=1e-3,
                         seed=9, stream_base=0, table_len=None, rng="philox", workers=1, epochs=1,
                         update=True, model=dm1, dim=D, trace_cap=0, schedule="dynamic")
    dm2 = DeviceModel.from_host(P.EmbeddingModel(base.copy(), np.zeros_like(base)))
    cfg = P.TrainingConfig(dim=D, window=5, negatives=5, subsample=1e-3, min_count=1, seed=9,
                           epochs=1, workers=1)
    st = StreamingTrainer(dm2, counts, cfg, float(off[-1]), 20_000, 2_000, syn.encoded.max_sentence_length(),
                          n_workers=1)
    cuts = [0, 100, 333, 334, 700, len(off) - 1]
    host_ids = torch.from_numpy(ids).pin_memory()
    chunks = [(host_ids[off[a]:off[b]], off[a:b + 1] - off[a], int(off[a])) for a, b in zip(cuts, cuts[1:])]
    res = list(st.train_chunks(chunks))
    assert sum(r[1] for r in res) == int(off[-1])
    assert sum(r[0] for r in res) == run.words_trained
    a, b = dm1.to_host(), dm2.to_host()
    np.testing.assert_allclose(b.input_vectors, a.input_vectors, rtol=0, atol=1e-6)
    np.testing.assert_allclose(b.output_vectors, a.output_vectors, rtol=0, atol=1e-6)


def test_streaming_after_launch_hook_is_stream_ordered():
    """train_chunks(after_launch=f) runs f between chunk i's kernel and chunk i+1's (the
    data-parallel average slot): model snapshots taken by the hook equal the state after
    training chunks 0..i one at a time."""
    P = _pkg()
    from paper_1604_04661_b200.synthetic import make_planted_corpus
    from paper_1604_04661_b200.model import DeviceModel
    from paper_1604_04661_b200.trainer import StreamingTrainer
    syn = make_planted_corpus(30_000, 400, n_clusters=4, cluster_size=5, sentence_len=29, seed=3)
    ids, off, counts = syn.encoded.ids, syn.encoded.offsets, syn.vocab.counts
    V, D = len(counts), 32
    base = np.random.default_rng(2).normal(size=(V, D)).astype(np.float32) * 0.1
    cfg = P.TrainingConfig(dim=D, window=4, negatives=5, subsample=1e-3, min_count=1, seed=5,
                           epochs=1, workers=1)
    cuts = [0, 200, 450, 700, len(off) - 1]
    host_ids = torch.from_numpy(ids).pin_memory()
    chunks = [(host_ids[off[a]:off[b]], off[a:b + 1] - off[a], int(off[a])) for a, b in zip(cuts, cuts[1:])]

    def trainer():
        dm = DeviceModel.from_host(P.EmbeddingModel(base.copy(), np.zeros_like(base)))
        return dm, StreamingTrainer(dm, counts, cfg, float(off[-1]), 20_000, 2_000,
                                    syn.encoded.max_sentence_length(), n_workers=1)
    dm1, st1 = trainer()
    want = []
    for c in chunks:
        st1.train_chunk(*c)
        want.append(dm1.m_out.clone())
    dm2, st2 = trainer()
    got = []
    res = list(st2.train_chunks(chunks, after_launch=lambda: got.append(dm2.m_out.clone())))
    assert len(res) == len(got) == len(chunks)
    for w, g in zip(want, got):
        torch.testing.assert_close(g, w, rtol=0, atol=1e-6)
