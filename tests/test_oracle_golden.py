"""Pin the C oracle against fixtures produced by the reference itself (CPU only).

Every fixture comes from tests/golden/make_golden.py running the reference
`sgns` package; a mismatch here means the oracle does not restate the
reference and no GPU parity claim built on it would hold.
"""

import numpy as np
import pytest

from helpers import TRACE_CASES, kernel_case, load_golden, trace_to_records, train_config

from oracle import oracle as O


def test_splitmix_stream_matches_reference():
    g = load_golden("rng")
    for i in range(int(g["n_cases"][0])):
        seed, stream = int(g[f"c{i}_seed"][0]), int(g[f"c{i}_stream"][0])
        st = O.new_state(seed, stream)
        assert st == int(g[f"c{i}_state0"][0])
        u, st = O.splitmix(st, 64)
        assert np.array_equal(u, g[f"c{i}_u64"])
        uni, st = O.splitmix(st, 64, "uniform")
        assert np.array_equal(uni, g[f"c{i}_uniform"])
        b7, st = O.splitmix(st, 64, "below", 7)
        assert np.array_equal(b7, g[f"c{i}_below7"])
        b8, st = O.splitmix(st, 64, "below", 100_000_000)
        assert np.array_equal(b8, g[f"c{i}_below1e8"])


def test_philox_known_answers():
    # Random123 known-answer vectors for philox4x32-10
    assert O.philox([0, 0, 0, 0], [0, 0]).tolist() == [0x6627E8D5, 0xE169C58D, 0xBC57AC4C, 0x9B00DBD8]
    assert O.philox([0xFFFFFFFF] * 4, [0xFFFFFFFF] * 2).tolist() == [
        0x408F276D, 0x41C83B0E, 0xA20BC7C6, 0x6D5451FD]
    assert O.philox([0x243F6A88, 0x85A308D3, 0x13198A2E, 0x03707344],
                    [0xA4093822, 0x299F31D0]).tolist() == [
        0xD16CFE09, 0x94FDCCEB, 0x5001E420, 0x24126EA1]


def test_sigmoid_table_index_rule():
    g = load_golden("tables")
    tab = g["sigmoid_f32"]
    got = np.array([O.sigmoid_table_f32(x, tab) for x in g["probe_x"]], dtype=np.float32)
    assert np.array_equal(got, g["probe_sig"])


def test_negative_table_boundaries():
    g = load_golden("tables")
    counts = g["kp_counts"]
    b = O.neg_boundaries(counts, 0.75, 100_003)
    slots = np.repeat(np.arange(len(counts), dtype=np.int32), np.diff(b, prepend=0))
    assert np.array_equal(slots, g["neg_small_slots"])
    big = O.neg_boundaries(g["neg_big_counts"], 0.75, 100_000_000)
    assert np.array_equal(np.diff(big, prepend=0), g["neg_big_slot_counts"])


def test_init_model():
    g = load_golden("init")
    for key in g.files:
        if not key.startswith("in64_"):
            continue
        _, V, D, seed = key.split("_")
        m = O.init_model(int(V), int(D), int(seed))
        assert np.array_equal(m, g[key])
        assert np.array_equal(m.astype(np.float32), g["in32_" + key[5:]])


@pytest.mark.parametrize("dtype", ["f64", "f32"])
def test_process_batch_naive_bitwise(dtype):
    g = load_golden("kernel")
    t = load_golden("tables")
    tab = t["sigmoid_f64"] if dtype == "f64" else t["sigmoid_f32"]
    npdt = np.float64 if dtype == "f64" else np.float32
    for i in range(int(g["n_cases"][0])):
        m_in, m_out, ins, outs, alpha, r_in, r_out = kernel_case(g, i)
        a, c = m_in.astype(npdt), m_out.astype(npdt)
        O.process_batch(a, c, ins, outs, alpha, tab)
        assert np.array_equal(a[r_in], g[f"c{i}_{dtype}_naive_min"]), i
        assert np.array_equal(c[r_out], g[f"c{i}_{dtype}_naive_mout"]), i
        # BLAS order is OpenBLAS's; the naive restatement stays within the reference's 2e-5
        np.testing.assert_allclose(a[r_in], g[f"c{i}_{dtype}_blas_min"], rtol=2e-5, atol=1e-7)
        np.testing.assert_allclose(c[r_out], g[f"c{i}_{dtype}_blas_mout"], rtol=2e-5, atol=1e-7)


def test_process_windows_is_sequential_process_batch():
    """The microbench CPU leg: one thread == the windows through process_batch in order;
    T threads on disjoint rows == the same result (no row is shared)."""
    rng = np.random.default_rng(5)
    V, D, K1 = 300, 24, 6
    tab = load_golden("tables")["sigmoid_f32"]
    m_in = rng.normal(size=(V, D)).astype(np.float32) * 0.3
    m_out = rng.normal(size=(V, D)).astype(np.float32) * 0.3
    ms = rng.integers(1, 11, size=40)
    off = np.concatenate([[0], np.cumsum(ms)]).astype(np.int32)
    ins = rng.integers(0, V, size=off[-1]).astype(np.int32)
    outs = rng.integers(0, V, size=(40, K1)).astype(np.int32)
    a, c = m_in.copy(), m_out.copy()
    for w in range(40):
        O.process_batch(a, c, ins[off[w]:off[w + 1]], outs[w], 0.025, tab)
    b, d = m_in.copy(), m_out.copy()
    O.process_windows(b, d, off, ins, outs, 0.025, tab, n_threads=1)
    assert np.array_equal(a, b) and np.array_equal(c, d)
    # disjoint rows: window w uses rows [w*7, w*7+7)
    ins2 = np.concatenate([np.arange(w * 7, w * 7 + 1) for w in range(40)]).astype(np.int32)
    off2 = np.arange(41, dtype=np.int32)
    outs2 = np.array([np.arange(w * 7 + 1, w * 7 + 7) for w in range(40)], np.int32)
    a, c = m_in.copy(), m_out.copy()
    O.process_windows(a, c, off2, ins2, outs2, 0.025, tab, n_threads=1)
    b, d = m_in.copy(), m_out.copy()
    O.process_windows(b, d, off2, ins2, outs2, 0.025, tab, n_threads=4)
    assert np.array_equal(a, b) and np.array_equal(c, d)


@pytest.mark.parametrize("case", TRACE_CASES, ids=[c[0] for c in TRACE_CASES])
def test_driver_stream_matches_reference_pipeline(case):
    """Windows, chunks and shared negatives: bit-exact vs subsample->iterate_windows->assemble_batches."""
    name, n, V, w, k, cap, dyn, sub, seed, stream, table_len = case
    g = load_golden("traces")
    ids, off, counts = g[f"{name}_ids"], g[f"{name}_offsets"], g[f"{name}_counts"]
    from paper_1604_04661_b200.corpus import default_table_length, keep_probabilities
    L = table_len or default_table_length(len(counts))
    slots = np.repeat(np.arange(len(counts), dtype=np.int32),
                      np.diff(O.neg_boundaries(counts, 0.75, L), prepend=0))
    keep = keep_probabilities(counts, int(counts.sum()), sub) if sub > 0 else None
    m = np.zeros((len(counts), 4), dtype=np.float32)
    expect = trace_to_records(g, name, cap, k + 1)
    run = O.OracleRun(ids, off, m, m.copy(), keep_probs=keep, window=w, negatives=k,
                      batch_cap=cap, dynamic=dyn, seed=seed, alpha0=0.025, floor_frac=1e-4,
                      total_x_epochs=float(off[-1]), epochs=1, loss_every=0, n_workers=1,
                      stream_base=stream, slots=slots, sig_table=np.zeros(1000, np.float32),
                      trace_cap=len(expect) + 10, update=False)
    run.run_to_completion()
    got, _ = run.worker_trace(0)
    assert got.shape == expect.shape
    assert np.array_equal(got, expect)
    assert run.workers[0].rng == int(g[f"{name}_final_state"][0])


def _oracle_train(name, threads=1):
    cfg = train_config(name)
    g = load_golden("train")
    t = load_golden("tables")
    from paper_1604_04661_b200.corpus import default_table_length, keep_probabilities
    ids, off, counts = g["ids"], g["offsets"], g["counts"]
    V, D = len(counts), cfg["dim"]
    dt = np.float64 if cfg["float64"] else np.float32
    m_in = O.init_model(V, D, cfg["seed"]).astype(dt)
    m_out = np.zeros((V, D), dtype=dt)
    slots = np.repeat(np.arange(V, dtype=np.int32),
                      np.diff(O.neg_boundaries(counts, 0.75, default_table_length(V)), prepend=0))
    keep = keep_probabilities(counts, int(counts.sum()), cfg["subsample"]) if cfg["subsample"] > 0 else None
    run = O.OracleRun(ids, off, m_in, m_out, keep_probs=keep, window=cfg["window"],
                      negatives=cfg["negatives"], batch_cap=cfg["batch_cap"],
                      dynamic=cfg["dynamic_window"], seed=cfg["seed"], alpha0=cfg["alpha0"],
                      floor_frac=1e-4, total_x_epochs=float(off[-1]) * cfg["epochs"],
                      epochs=cfg["epochs"], loss_every=cfg["loss_sample_every"],
                      n_workers=threads, slots=slots,
                      sig_table=t["sigmoid_f64"] if dt == np.float64 else t["sigmoid_f32"])
    run.run_to_completion()
    return run, g


@pytest.mark.parametrize("name", ["f64_naive", "f32_naive", "f64_cap1_k1", "f64_w10_cap4",
                                  "f64_static_nosub", "f32_k15_loss1", "f64_loss7"])
def test_fused_driver_bitwise_vs_reference_train_encoded(name):
    run, g = _oracle_train(name)
    assert np.array_equal(run.m_in, g[f"{name}_min"])
    assert np.array_equal(run.m_out, g[f"{name}_mout"])
    trained, read, loss = run.stats()
    assert [trained, read] == g[f"{name}_stats"].tolist()
    np.testing.assert_allclose(loss, g[f"{name}_loss"], rtol=1e-12)
    shared_read = int(run.shared[0])
    alpha = max(1.0 - shared_read / (float(g["offsets"][-1]) * train_config(name)["epochs"] + 1.0), 1e-4) * 0.025
    assert alpha == pytest.approx(float(g[f"{name}_final_alpha"][0]), rel=1e-12)


def test_fused_driver_f32_blas_within_tolerance():
    """The reference's float32 default is BLAS (unrestatable summation order): loss within 0.1%."""
    run, g = _oracle_train("f32_blas")
    trained, read, loss = run.stats()
    assert [trained, read] == g["f32_blas_stats"].tolist()
    np.testing.assert_allclose(loss, g["f32_blas_loss"], rtol=1e-3)
    np.testing.assert_allclose(run.m_in, g["f32_blas_min"], rtol=0, atol=5e-3)
