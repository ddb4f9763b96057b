"""Host-side corpus formats on either side of the device path.

These are the data structures the reference's training entry points accept
(`sgns/corpus.py`), restated so a caller of the reference can hand the same
objects to this package.  Nothing here is on the hot path: the device driver
(`csrc/sgns_fast.cuh`, `csrc/sgns_kernels.cu`) consumes `EncodedCorpus.ids` / `.offsets` once they
are resident in HBM, and the two samplers are built here (float64, host) and
uploaded once per run.

Reference map:
  Vocabulary / keep_probs        sgns/corpus.py:36-83
  build_vocab                    sgns/corpus.py:86-105
  keep_probability               sgns/corpus.py:108-117
  default_table_length           sgns/corpus.py:132-136
  build_negative_table           sgns/corpus.py:139-155  (slot boundaries only;
                                 the 10^8-slot array itself is expanded on device)
  EncodedCorpus / encode_corpus  sgns/corpus.py:243-311
  partition_sentences            sgns/corpus.py:314-334
  split_by_tokens                sgns/trainer.py:314-329
"""

from __future__ import annotations

import math
from dataclasses import dataclass
from typing import Iterable, Iterator

import numpy as np

MAX_SENTENCE_TOKENS = 1000
# Device workers stage one subsampled sentence at a time; the reference's own
# per-thread buffer has the same bound (sgns/trainer.py:377).
KEPT_BUFFER_TOKENS = 1024
NEGATIVE_POWER = 0.75
FULL_TABLE_LENGTH = 100_000_000


class EmptyVocabularyError(ValueError):
    """No token survived the min_count filter."""


class TableLengthError(ValueError):
    """Requested negative-table length is smaller than the vocabulary."""


class PartitionError(ValueError):
    """Corpus cannot be split into the requested number of shards."""


@dataclass
class Vocabulary:
    """Word ids ordered by descending count, ties by first occurrence."""

    tokens: list[str]
    counts: np.ndarray  # int64 per id
    index: dict[str, int]
    total_tokens: int

    @property
    def size(self) -> int:
        return len(self.tokens)

    def __len__(self) -> int:
        return len(self.tokens)

    def __contains__(self, token: str) -> bool:
        return token in self.index

    def keep_probs(self, threshold: float) -> np.ndarray:
        """Per-id keep probability, float64 (same arithmetic as keep_probability)."""
        return keep_probabilities(self.counts, self.total_tokens, threshold)

    def save(self, path: str) -> None:
        with open(path, "w", encoding="utf-8") as fh:
            for token, count in zip(self.tokens, self.counts):
                fh.write(f"{token}\t{int(count)}\n")

    @classmethod
    def load(cls, path: str) -> "Vocabulary":
        tokens: list[str] = []
        counts: list[int] = []
        with open(path, encoding="utf-8") as fh:
            for line in fh:
                token, _, count = line.rstrip("\n").partition("\t")
                tokens.append(token)
                counts.append(int(count))
        if not tokens:
            raise EmptyVocabularyError(f"no vocabulary entries in {path}")
        return cls(tokens, np.asarray(counts, dtype=np.int64),
                   {t: i for i, t in enumerate(tokens)}, int(sum(counts)))

    @classmethod
    def from_counts(cls, counts: np.ndarray, names: list[str] | None = None) -> "Vocabulary":
        """Vocabulary over already-ordered ids 0..V-1 (synthetic corpora)."""
        counts = np.asarray(counts, dtype=np.int64)
        if names is None:
            names = [f"w{i}" for i in range(len(counts))]
        return cls(list(names), counts, {t: i for i, t in enumerate(names)},
                   int(counts.sum()))


def build_vocab(token_stream: Iterable[str], min_count: int) -> Vocabulary:
    """Count tokens; keep count >= min_count; order by count desc, first occurrence."""
    counts: dict[str, int] = {}
    for token in token_stream:
        counts[token] = counts.get(token, 0) + 1
    # dicts keep first-occurrence order and sorted() is stable, so ties stay put
    kept = sorted(((t, c) for t, c in counts.items() if c >= min_count),
                  key=lambda tc: -tc[1])
    if not kept:
        raise EmptyVocabularyError(
            f"no token appears at least min_count={min_count} times")
    tokens = [t for t, _ in kept]
    arr = np.fromiter((c for _, c in kept), dtype=np.int64, count=len(kept))
    return Vocabulary(tokens, arr, {t: i for i, t in enumerate(tokens)}, int(arr.sum()))


def keep_probability(word_frequency_fraction: float, threshold: float) -> float:
    """p = (sqrt(f/t) + 1) * (t/f), clamped to 1."""
    f, t = word_frequency_fraction, threshold
    return min(1.0, (math.sqrt(f / t) + 1.0) * (t / f))


def keep_probabilities(counts: np.ndarray, total: int, threshold: float) -> np.ndarray:
    """Vectorised keep_probability; IEEE sqrt/div make it bit-identical per element."""
    f = np.asarray(counts, dtype=np.int64) / float(total)
    t = float(threshold)
    return np.minimum(1.0, (np.sqrt(f / t) + 1.0) * (t / f))


def default_table_length(vocab_size: int) -> int:
    if vocab_size >= 10_000:
        return FULL_TABLE_LENGTH
    return max(vocab_size, 10_000 * vocab_size)


@dataclass
class NegativeTable:
    """Unigram^power slot table, kept as per-word slot boundaries.

    Word w owns slots [boundaries[w-1], boundaries[w]).  The device expands
    this into the reference's int32 slot array once per run (`slots()` does
    the same on host, for small tables and tests).
    """

    boundaries: np.ndarray  # int64, len V, boundaries[-1] == length
    power: float
    source_vocab_size: int

    @property
    def length(self) -> int:
        return int(self.boundaries[-1])

    def __len__(self) -> int:
        return self.length

    def slot_counts(self) -> np.ndarray:
        return np.diff(self.boundaries, prepend=0)

    def slots(self) -> np.ndarray:
        return np.repeat(np.arange(self.source_vocab_size, dtype=np.int32), self.slot_counts())


def negative_table_boundaries(counts: np.ndarray, power: float, length: int) -> np.ndarray:
    """floor(L * cumsum(count^power) / total), last forced to L (float64, as the reference)."""
    weights = np.power(np.asarray(counts).astype(np.float64), power)
    cumulative = np.cumsum(weights)
    bounds = np.floor(length * cumulative / cumulative[-1]).astype(np.int64)
    bounds[-1] = length
    return bounds


def build_negative_table(vocab: Vocabulary, power: float = NEGATIVE_POWER,
                         length: int | None = None) -> NegativeTable:
    if length is None:
        length = default_table_length(vocab.size)
    if length < vocab.size:
        raise TableLengthError(
            f"table length {length} is smaller than vocabulary size {vocab.size}")
    return NegativeTable(negative_table_boundaries(vocab.counts, power, length),
                         power, vocab.size)


@dataclass
class EncodedCorpus:
    """Flat int32 ids plus int64 sentence offsets (sentence i = ids[off[i]:off[i+1]])."""

    ids: np.ndarray
    offsets: np.ndarray
    sentence_bytes: np.ndarray

    @property
    def n_sentences(self) -> int:
        return len(self.offsets) - 1

    @property
    def n_tokens(self) -> int:
        return int(self.offsets[-1])

    def sentence(self, i: int) -> np.ndarray:
        return self.ids[self.offsets[i]:self.offsets[i + 1]]

    def max_sentence_length(self) -> int:
        if self.n_sentences == 0:
            return 0
        return int(np.diff(self.offsets).max())


def read_tokens(path: str) -> Iterator[str]:
    with open(path, encoding="utf-8") as fh:
        for line in fh:
            yield from line.split()


def encode_corpus(path: str, vocab: Vocabulary,
                  max_sentence: int = MAX_SENTENCE_TOKENS) -> EncodedCorpus:
    """Lines are sentences; OOV tokens dropped; long lines split every max_sentence ids."""
    chunks: list[np.ndarray] = []
    offsets = [0]
    sent_bytes: list[int] = []
    index = vocab.index
    with open(path, encoding="utf-8") as fh:
        for line in fh:
            current: list[int] = []
            nbytes = 0
            for token in line.split():
                nbytes += len(token.encode("utf-8")) + 1
                wid = index.get(token)
                if wid is None:
                    continue
                current.append(wid)
                if len(current) >= max_sentence:
                    chunks.append(np.asarray(current, dtype=np.int32))
                    offsets.append(offsets[-1] + len(current))
                    sent_bytes.append(nbytes)
                    current, nbytes = [], 0
            if current:
                chunks.append(np.asarray(current, dtype=np.int32))
                offsets.append(offsets[-1] + len(current))
                sent_bytes.append(nbytes)
    flat = np.concatenate(chunks) if chunks else np.empty(0, dtype=np.int32)
    return EncodedCorpus(flat, np.asarray(offsets, dtype=np.int64),
                         np.asarray(sent_bytes, dtype=np.int64))


def partition_sentences(encoded: EncodedCorpus, n_parts: int) -> list[tuple[int, int]]:
    """n contiguous, non-empty sentence ranges of near-equal byte size."""
    if n_parts < 1:
        raise PartitionError("need at least one shard")
    n = encoded.n_sentences
    if n_parts > n:
        raise PartitionError(f"cannot split {n} sentences into {n_parts} shards")
    cum = np.cumsum(encoded.sentence_bytes)
    total = float(cum[-1])
    bounds = [0]
    for k in range(1, n_parts):
        cut = int(np.searchsorted(cum, total * k / n_parts)) + 1
        bounds.append(max(bounds[-1] + 1, min(cut, n - (n_parts - k))))
    bounds.append(n)
    return [(bounds[i], bounds[i + 1]) for i in range(n_parts)]


def split_by_tokens(offsets: np.ndarray, sent_lo: int, sent_hi: int,
                    parts: int) -> list[tuple[int, int]]:
    """Contiguous sentence sub-ranges with near-equal token counts (may be empty)."""
    base = offsets[sent_lo]
    tokens = np.asarray(offsets[sent_lo + 1:sent_hi + 1]) - base
    total = float(tokens[-1]) if len(tokens) else 0.0
    if parts <= 0:
        raise ValueError("parts must be >= 1")
    # searchsorted over all cut targets at once; identical to the per-k loop
    targets = total * np.arange(1, parts, dtype=np.float64) / parts
    cuts = sent_lo + np.searchsorted(tokens, targets) + 1
    bounds = np.empty(parts + 1, dtype=np.int64)
    bounds[0] = sent_lo
    prev = sent_lo
    for k, cut in enumerate(cuts, start=1):
        prev = min(max(int(cut), prev), sent_hi)
        bounds[k] = prev
    bounds[parts] = sent_hi
    return [(int(bounds[i]), int(bounds[i + 1])) for i in range(parts)]


# ---------------------------------------------------------------- native ingestion ----
def _threads(threads: int | None) -> int:
    import os
    return threads if threads else max(1, len(os.sched_getaffinity(0)))


def _native_vocab_to_python(L, handle, n: int, nbytes: int) -> Vocabulary:
    import ctypes as C
    blob = C.create_string_buffer(max(nbytes, 1))
    offs = np.empty(n + 1, dtype=np.int64)
    counts = np.empty(n, dtype=np.int64)
    if L.sgns_vocab_export(handle, blob, offs.ctypes.data, counts.ctypes.data) != 0:
        raise RuntimeError("sgns_vocab_export failed")
    raw = blob.raw
    tokens = [raw[offs[i]:offs[i + 1]].decode("utf-8") for i in range(n)]
    return Vocabulary(tokens, counts, {t: i for i, t in enumerate(tokens)}, int(counts.sum()))


def build_vocab_file(path: str, min_count: int, threads: int | None = None) -> Vocabulary:
    """build_vocab(read_tokens(path), min_count), computed by the multithreaded C++ scanner."""
    import ctypes as C
    from . import _lib
    L = _lib.lib()
    h, n, nb = C.c_void_p(), C.c_int64(), C.c_int64()
    rc = L.sgns_vocab_build(path.encode(), min_count, _threads(threads), C.byref(h), C.byref(n), C.byref(nb))
    if rc == -6:
        raise EmptyVocabularyError(f"no token appears at least min_count={min_count} times")
    if rc == -5:
        raise FileNotFoundError(path)
    if rc != 0:
        raise ValueError(f"sgns_vocab_build failed ({rc})")
    try:
        return _native_vocab_to_python(L, h, n.value, nb.value)
    finally:
        L.sgns_vocab_free(h)


def encode_corpus_file(path: str, vocab: Vocabulary, max_sentence: int = MAX_SENTENCE_TOKENS,
                       threads: int | None = None) -> EncodedCorpus:
    """encode_corpus(path, vocab), computed by the multithreaded C++ scanner."""
    import ctypes as C
    from . import _lib
    L = _lib.lib()
    enc_tokens = [t.encode("utf-8") for t in vocab.tokens]
    offs = np.zeros(len(enc_tokens) + 1, dtype=np.int64)
    offs[1:] = np.cumsum([len(t) for t in enc_tokens])
    blob = b"".join(enc_tokens)
    blob_buf = C.create_string_buffer(blob, max(len(blob), 1))
    counts = np.ascontiguousarray(vocab.counts, dtype=np.int64)
    vh = C.c_void_p()
    if L.sgns_vocab_from_tokens(C.addressof(blob_buf), offs.ctypes.data, counts.ctypes.data,
                                len(enc_tokens), C.byref(vh)) != 0:
        raise ValueError("sgns_vocab_from_tokens failed")
    try:
        eh, nt, ns = C.c_void_p(), C.c_int64(), C.c_int64()
        rc = L.sgns_encode(vh, path.encode(), max_sentence, _threads(threads), C.byref(eh),
                           C.byref(nt), C.byref(ns))
        if rc == -5:
            raise FileNotFoundError(path)
        if rc != 0:
            raise ValueError(f"sgns_encode failed ({rc})")
        try:
            ids = np.empty(nt.value, dtype=np.int32)
            offsets = np.empty(ns.value + 1, dtype=np.int64)
            sbytes = np.empty(ns.value, dtype=np.int64)
            L.sgns_encoded_export(eh, ids.ctypes.data, offsets.ctypes.data, sbytes.ctypes.data)
        finally:
            L.sgns_encoded_free(eh)
    finally:
        L.sgns_vocab_free(vh)
    return EncodedCorpus(ids, offsets, sbytes)
