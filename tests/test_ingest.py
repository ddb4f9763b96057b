"""Native corpus ingestion (C++) against the reference's own
build_vocab(read_tokens(path)) / encode_corpus(path, vocab) outputs on a text file
exercising every str.split() whitespace class, universal newlines, >1000-token lines,
OOV-only and empty lines and an unterminated last line.  Host code only (no GPU)."""

import os

import numpy as np
import pytest

from helpers import GOLDEN, load_golden

from paper_1604_04661_b200.corpus import (EmptyVocabularyError, build_vocab, build_vocab_file,
                                          encode_corpus, encode_corpus_file, read_tokens)

PATH = os.path.join(GOLDEN, "ingest_corpus.txt")


@pytest.mark.parametrize("threads", [1, 3, 8])
def test_native_vocab_and_encoding_match_reference(threads):
    g = load_golden("ingest")
    voc = build_vocab_file(PATH, 2, threads=threads)
    assert voc.tokens == str(g["tokens"]).split("\x00")
    assert np.array_equal(voc.counts, g["counts"])
    assert voc.total_tokens == int(g["total"][0])
    assert all(voc.index[t] == i for i, t in enumerate(voc.tokens))
    enc = encode_corpus_file(PATH, voc, threads=threads)
    assert np.array_equal(enc.ids, g["ids"])
    assert np.array_equal(enc.offsets, g["offsets"])
    assert np.array_equal(enc.sentence_bytes, g["sentence_bytes"])


def test_python_restatement_matches_reference_too():
    g = load_golden("ingest")
    voc = build_vocab(read_tokens(PATH), 2)
    assert voc.tokens == str(g["tokens"]).split("\x00")
    enc = encode_corpus(PATH, voc)
    assert np.array_equal(enc.ids, g["ids"]) and np.array_equal(enc.sentence_bytes, g["sentence_bytes"])


def test_native_errors(tmp_path):
    with pytest.raises(FileNotFoundError):
        build_vocab_file(str(tmp_path / "missing.txt"), 1)
    p = tmp_path / "few.txt"
    p.write_text("a b c\n", encoding="utf-8")
    with pytest.raises(EmptyVocabularyError):
        build_vocab_file(str(p), 2)
    e = tmp_path / "empty.txt"
    e.write_text("", encoding="utf-8")
    with pytest.raises(EmptyVocabularyError):
        build_vocab_file(str(e), 1)


def test_native_matches_python_on_synthetic_text(tmp_path):
    from paper_1604_04661_b200.synthetic import make_planted_corpus
    syn = make_planted_corpus(200_000, 3000, n_clusters=5, cluster_size=10, seed=4)
    path = str(tmp_path / "syn.txt")
    syn.write_text(path)
    a = build_vocab_file(path, 3, threads=4)
    b = build_vocab(read_tokens(path), 3)
    assert a.tokens == b.tokens and np.array_equal(a.counts, b.counts)
    ea, eb = encode_corpus_file(path, a, threads=5), encode_corpus(path, b)
    assert np.array_equal(ea.ids, eb.ids) and np.array_equal(ea.offsets, eb.offsets)
    assert np.array_equal(ea.sentence_bytes, eb.sentence_bytes)
