"""CPU-only tests: host logic against reference fixtures, the C-ABI library's
exports (loaded, no device calls), the alias table, and the synthetic corpora."""

import os
import re

import numpy as np
import pytest

from helpers import ROOT, load_golden

import paper_1604_04661_b200 as P
from paper_1604_04661_b200 import _lib
from paper_1604_04661_b200.corpus import (EncodedCorpus, default_table_length, keep_probabilities,
                                          negative_table_boundaries, partition_sentences,
                                          split_by_tokens)
from paper_1604_04661_b200.distributed import row_runs, select_sync_rows, sync_row_ranges
from paper_1604_04661_b200.rng import new_state


def test_library_exports_every_header_symbol():
    header = open(os.path.join(ROOT, "include", "sgns_b200.h")).read()
    declared = set(re.findall(r"\b(sgns_[a-z0-9_]+)\s*\(", header))
    assert declared == set(_lib.EXPORTED)
    L = _lib.lib()
    for sym in declared:
        assert getattr(L, sym) is not None
    assert L.sgns_abi_version() == 2
    assert L.sgns_error_string(-3).decode().startswith("per-warp")


def test_device_entry_points_validate_before_launch():
    L = _lib.lib()
    assert L.sgns_update_windows(0, None, None, None, None, 1, 4, 4, None, None, None, 1, 2, 1,
                                 None, None, 0, 0, None, None, None, None) == -1
    assert L.sgns_update_windows(0, None, None, None, None, 1, 4, 4, None, None, None, 0, 2, 1,
                                 None, None, 0, 0, None, None, None, None) == 0  # empty batch
    assert L.sgns_drive(None, None) == -1
    assert L.sgns_init_model(0, None, None, 1, 4, 4, 0, None) == -1
    assert L.sgns_init_model(0, 1, 1, 1, 3, 3, 0, None) == -2  # row not a multiple of 16 bytes


def test_rng_new_state_matches_reference():
    g = load_golden("rng")
    for i in range(int(g["n_cases"][0])):
        assert new_state(int(g[f"c{i}_seed"][0]), int(g[f"c{i}_stream"][0])) == int(g[f"c{i}_state0"][0])


def test_keep_probs_and_negative_table_match_reference():
    t = load_golden("tables")
    counts = t["kp_counts"]
    for th in (1e-3, 1e-4, 1e-5):
        assert np.array_equal(keep_probabilities(counts, int(counts.sum()), th), t[f"kp_{th:g}"])
    b = negative_table_boundaries(counts, 0.75, 100_003)
    assert np.array_equal(np.repeat(np.arange(len(counts)), np.diff(b, prepend=0)), t["neg_small_slots"])
    big = negative_table_boundaries(t["neg_big_counts"], 0.75, 100_000_000)
    assert np.array_equal(np.diff(big, prepend=0), t["neg_big_slot_counts"])
    for V in (1, 9_999, 10_000, 250_000):
        assert default_table_length(V) == int(t[f"deflen_{V}"][0])
    assert np.array_equal(P.model.SIGMOID_TABLE_F32, t["sigmoid_f32"])
    assert np.array_equal(P.model.SIGMOID_TABLE_F64, t["sigmoid_f64"])


def test_sync_rows_partition_split_match_reference():
    d = load_golden("dist")
    for k in range(int(d["n_sync"][0])):
        V, hot, rot, period = d[f"s{k}_args"].tolist()
        pol = P.SyncPolicy(hot_rows=None if hot < 0 else hot, rotation_chunk=None if rot < 0 else rot)
        rows = select_sync_rows(V, pol, period)
        assert len(rows) == int(d[f"s{k}_len"][0])
        assert [list(r) for r in row_runs(rows)] == d[f"s{k}_runs"].tolist()
        assert len(sync_row_ranges(V, pol, period)) <= 2
    g = load_golden("train")
    enc = EncodedCorpus(g["ids"], g["offsets"], g["sentence_bytes"])
    for n in (1, 2, 3, 8):
        assert partition_sentences(enc, n) == [tuple(x) for x in d[f"part_{n}"].tolist()]
        assert split_by_tokens(enc.offsets, 0, enc.n_sentences, n) == [tuple(x) for x in d[f"split_{n}"].tolist()]
        lo, hi = partition_sentences(enc, 2)[1]
        assert split_by_tokens(enc.offsets, lo, hi, n) == [tuple(x) for x in d[f"split_sub_{n}"].tolist()]
    assert split_by_tokens(enc.offsets, 0, enc.n_sentences, 700) == [tuple(x) for x in d["split_big"].tolist()]
    assert P.scaled_alpha0(0.025, 4) == pytest.approx(0.05)


@pytest.mark.parametrize("V,seed", [(2, 0), (7, 1), (100, 2), (5000, 3)])
def test_alias_table_encodes_unigram_power_exactly(V, seed):
    """The alias table's implied distribution equals count^0.75 / sum to ~1e-9 (host C++ in the .so)."""
    rng = np.random.default_rng(seed)
    counts = rng.integers(1, 1_000_000, size=V).astype(np.int64)
    thr = np.empty(V, np.uint32)
    idx = np.empty(V, np.int32)
    assert _lib.lib().sgns_build_alias(counts.ctypes.data, V, 0.75, thr.ctypes.data, idx.ctypes.data) == 0
    p_keep = thr.astype(np.float64) / 2.0**32
    full = thr == 0xFFFFFFFF
    p_keep[full] = 1.0
    implied = p_keep.copy()
    np.add.at(implied, idx, np.where(full, 0.0, 1.0 - p_keep))
    implied /= V
    w = counts.astype(np.float64) ** 0.75
    np.testing.assert_allclose(implied, w / w.sum(), rtol=1e-6, atol=1e-9)


def test_config_validation():
    P.TrainingConfig().validate()
    for field, value in [("dim", 0), ("window", 0), ("negatives", 0), ("epochs", 0), ("threads", 0),
                         ("batch_cap", 0), ("alpha0", -1.0), ("alpha_floor_fraction", 1.5),
                         ("kernel", "gpu"), ("matmul", "magic"), ("rng", "mt"), ("workers", 0),
                         ("negatives", 40)]:
        with pytest.raises(P.ConfigError):
            P.TrainingConfig(**{field: value}).validate()


def test_update_alpha_schedule():
    assert P.update_alpha(0, 1000.0, 0.025, 1e-4) == pytest.approx(0.025)
    assert P.update_alpha(10**6, 1e6, 0.025, 1e-4) == pytest.approx(0.025 * 1e-4)


def test_planted_corpus_vocabulary_order():
    from paper_1604_04661_b200.synthetic import make_planted_corpus
    syn = make_planted_corpus(50_000, 2_000, n_clusters=5, cluster_size=8, sentence_len=50, seed=3)
    c = syn.vocab.counts
    assert (np.diff(c) <= 0).all()
    assert np.array_equal(np.bincount(syn.encoded.ids, minlength=len(c)), c)
    # ties broken by first occurrence
    first = np.full(len(c), len(syn.encoded.ids))
    np.minimum.at(first, syn.encoded.ids, np.arange(len(syn.encoded.ids)))
    for v in np.unique(c):
        grp = np.flatnonzero(c == v)
        assert (np.diff(first[grp]) > 0).all()
    assert all(len(cl) == 8 for cl in syn.clusters)


def test_eval_similarity_matches_reference():
    from paper_1604_04661_b200.evaluate import similarity_score
    e = load_golden("eval")
    import tempfile
    with tempfile.NamedTemporaryFile("w", suffix=".txt", delete=False) as fh:
        fh.write(str(e["pairs"][0]))
        path = fh.name
    names = [f"w{i}" for i in range(len(e["counts"]))]  # any index works: pairs use vocab names
    from paper_1604_04661_b200.synthetic import make_planted_corpus
    syn = make_planted_corpus(20_000, 500, n_clusters=6, cluster_size=8, seed=9)
    rho, used, skipped = similarity_score(e["vecs"], syn.vocab.index, path)
    os.unlink(path)
    assert [used, skipped] == e["rho"][1:].astype(int).tolist()
    assert rho == pytest.approx(float(e["rho"][0]), abs=1e-9)
    del names


def test_sampler_rejects_tables_without_a_second_word():
    """A negative table with one distinct word would make the target-rejection loop spin
    forever on the device (the reference hangs the same way); refuse it up front."""
    from paper_1604_04661_b200.trainer import DeviceSampler
    with pytest.raises(ValueError):
        DeviceSampler(np.array([7, 0, 0]), "philox", device="cpu")
    with pytest.raises(ValueError):
        DeviceSampler(np.array([5, 0]), "splitmix", table_length=10, device="cpu")


def test_row_stride_policy():
    """model.py padded_ld: whole 32-byte sectors; float32 rows on whole 128-byte lines when
    that costs at most 12.5% (DESIGN 2)."""
    from paper_1604_04661_b200.model import padded_ld
    f32 = {300: 320, 200: 224, 100: 104, 128: 128, 4: 8, 7: 8, 64: 64, 512: 512, 500: 512, 33: 40, 29: 32}
    for dim, ld in f32.items():
        assert padded_ld(dim, np.float32) == ld, (dim, padded_ld(dim, np.float32))
        assert ld >= dim and ld % 8 == 0
    for dim, ld in {300: 300, 5: 8, 101: 104}.items():
        assert padded_ld(dim, np.float64) == ld
