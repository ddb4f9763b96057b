"""Property tests (hypothesis) of the host logic around the device path, in the style of
the reference's own (tests/test_corpus.py:116-134, :278-301)."""

import numpy as np
import pytest
from hypothesis import given, settings, strategies as st

from paper_1604_04661_b200 import _lib
from paper_1604_04661_b200.corpus import (EncodedCorpus, PartitionError, build_vocab, build_vocab_file,
                                          encode_corpus, encode_corpus_file, keep_probabilities,
                                          negative_table_boundaries, partition_sentences, read_tokens,
                                          split_by_tokens)
from paper_1604_04661_b200.distributed import SyncPolicy, select_sync_rows

lengths = st.lists(st.integers(1, 60), min_size=1, max_size=80)


@given(lengths, st.integers(1, 12))
@settings(max_examples=60, deadline=None)
def test_split_by_tokens_contiguous_cover_balanced(lens, parts):
    off = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    r = split_by_tokens(off, 0, len(lens), parts)
    assert len(r) == parts and r[0][0] == 0 and r[-1][1] == len(lens)
    assert all(a[1] == b[0] for a, b in zip(r, r[1:]))
    sizes = [off[b] - off[a] for a, b in r]
    assert max(sizes) <= off[-1] / parts + max(lens) + 1e-9


@given(lengths, st.integers(1, 12))
@settings(max_examples=60, deadline=None)
def test_partition_nonempty_contiguous(lens, n):
    off = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    enc = EncodedCorpus(np.zeros(off[-1], np.int32), off, np.array(lens, dtype=np.int64) * 3)
    if n > len(lens):
        with pytest.raises(PartitionError):
            partition_sentences(enc, n)
        return
    r = partition_sentences(enc, n)
    assert r[0][0] == 0 and r[-1][1] == len(lens) and all(b > a for a, b in r)
    assert all(a[1] == b[0] for a, b in zip(r, r[1:]))


@given(st.lists(st.integers(1, 10**6), min_size=1, max_size=200), st.integers(0, 3))
@settings(max_examples=60, deadline=None)
def test_negative_table_share_within_one_slot(counts, extra):
    counts = np.array(counts, dtype=np.int64)
    L = len(counts) * (10 + extra * 1000)
    b = negative_table_boundaries(counts, 0.75, L)
    share = np.diff(b, prepend=0)
    w = counts.astype(np.float64) ** 0.75
    assert b[-1] == L and (share >= 0).all()
    assert np.abs(share - L * w / w.sum()).max() <= 1.0 + 1e-6


@given(st.lists(st.integers(1, 10**6), min_size=1, max_size=300))
@settings(max_examples=60, deadline=None)
def test_alias_table_distribution_exact(counts):
    counts = np.array(counts, dtype=np.int64)
    V = len(counts)
    thr = np.empty(V, np.uint32)
    idx = np.empty(V, np.int32)
    assert _lib.lib().sgns_build_alias(counts.ctypes.data, V, 0.75, thr.ctypes.data, idx.ctypes.data) == 0
    keep = np.where(thr == 0xFFFFFFFF, 1.0, thr / 2.0**32)
    implied = keep.copy()
    np.add.at(implied, idx, np.where(thr == 0xFFFFFFFF, 0.0, 1.0 - keep))
    w = counts.astype(np.float64) ** 0.75
    np.testing.assert_allclose(implied / V, w / w.sum(), rtol=1e-6, atol=1e-9)


@given(st.lists(st.integers(1, 10**7), min_size=2, max_size=100), st.sampled_from([1e-3, 1e-4, 1e-5]))
@settings(max_examples=50, deadline=None)
def test_keep_probability_monotone(counts, t):
    c = np.sort(np.array(counts, dtype=np.int64))
    p = keep_probabilities(c, int(c.sum()), t)
    assert ((p > 0) & (p <= 1)).all() and (np.diff(p) <= 1e-15).all()


@given(st.integers(1, 5000), st.integers(0, 200), st.integers(0, 300))
@settings(max_examples=60, deadline=None)
def test_sync_rows_hot_always_and_full_coverage(V, hot, rot):
    hot = min(hot, V)
    rot = min(rot, V - hot)
    pol = SyncPolicy(hot_rows=hot, rotation_chunk=rot)
    seen = set()
    n_chunks = -(-(V - hot) // rot) if rot else 1
    for period in range(n_chunks):
        r = select_sync_rows(V, pol, period)
        assert set(range(hot)) <= set(r.tolist())
        seen |= set(r.tolist())
    if rot:
        assert seen == set(range(V))


ws = st.sampled_from([" ", "  ", "\t", "\x0b", "\x0c", "\x1c", "\xa0", " ", "　", "\x85"])
nl = st.sampled_from(["\n", "\r\n", "\r"])
word = st.sampled_from(["a", "bb", "c", "dé", "日", "A", "x​y", "zz"])


@given(st.lists(st.tuples(st.lists(st.tuples(word, ws), max_size=12), nl), min_size=1, max_size=30),
       st.integers(1, 3), st.integers(1, 4))
@settings(max_examples=60, deadline=None)
def test_native_ingestion_equals_python(tmp_path_factory, lines, min_count, max_sentence):
    text = "".join("".join(w + s for w, s in toks) + e for toks, e in lines)
    path = tmp_path_factory.mktemp("ing") / "c.txt"
    path.write_text(text, encoding="utf-8", newline="")
    try:
        ref = build_vocab(read_tokens(str(path)), min_count)
    except ValueError:
        with pytest.raises(ValueError):
            build_vocab_file(str(path), min_count, threads=3)
        return
    got = build_vocab_file(str(path), min_count, threads=3)
    assert got.tokens == ref.tokens and np.array_equal(got.counts, ref.counts)
    a = encode_corpus_file(str(path), got, max_sentence=max_sentence, threads=2)
    b = encode_corpus(str(path), ref, max_sentence=max_sentence)
    assert np.array_equal(a.ids, b.ids) and np.array_equal(a.offsets, b.offsets)
    assert np.array_equal(a.sentence_bytes, b.sentence_bytes)
