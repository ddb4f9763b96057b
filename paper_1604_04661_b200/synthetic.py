"""Seeded synthetic corpora standing in for text8 / the 1B-word benchmark.

BASELINE.json's configs name seeded Zipf corpora with planted clusters; the
reference only ships a plain Zipf generator (`tests/conftest.py:49-66`) and a
topic-only one (`tests/conftest.py:69-90`), so this module combines them:
Zipf(s) background tokens, plus short same-cluster runs overwritten into
sentences so that cluster members co-occur within a window.  The corpus is
emitted directly as int32 ids in the reference's vocabulary order (count
descending, ties by first occurrence, `sgns/corpus.py:95-97`) together with a
`Vocabulary`, so both this package and the reference's `train_encoded` can be
fed the same arrays without text ingestion.  Gold similarity pairs follow
`tests/test_acceptance.py:454-467` (within-cluster high, cross-cluster low).

No dataset items are reproduced: every token is "w<raw id>".
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .corpus import EncodedCorpus, Vocabulary


@dataclass
class SyntheticCorpus:
    vocab: Vocabulary
    encoded: EncodedCorpus
    clusters: list[np.ndarray]  # final vocabulary ids of each planted cluster
    seed: int

    def gold_pairs(self, pairs_per_cluster: int = 8, seed: int = 1,
                   partner_offset: int = 3) -> list[tuple[str, str, float]]:
        rng = np.random.default_rng(seed)
        names = self.vocab.tokens
        out: list[tuple[str, str, float]] = []
        n = len(self.clusters)
        for t, words in enumerate(self.clusters):
            other = self.clusters[(t + partner_offset) % n]
            for _ in range(pairs_per_cluster):
                a, b = rng.choice(len(words), size=2, replace=False)
                out.append((names[words[a]], names[words[b]],
                            round(float(rng.uniform(7.5, 9.5)), 2)))
            for _ in range(pairs_per_cluster):
                out.append((names[words[rng.integers(len(words))]],
                            names[other[rng.integers(len(other))]],
                            round(float(rng.uniform(0.5, 2.5)), 2)))
        return out

    def write_gold_pairs(self, path: str, **kw) -> None:
        with open(path, "w", encoding="utf-8") as fh:
            for a, b, s in self.gold_pairs(**kw):
                fh.write(f"{a} {b} {s:.2f}\n")

    def write_text(self, path: str) -> None:
        """One line per sentence, tokens as vocabulary names (for text-path APIs)."""
        names = np.asarray(self.vocab.tokens, dtype=object)
        off = self.encoded.offsets
        with open(path, "w", encoding="utf-8") as fh:
            for s in range(self.encoded.n_sentences):
                fh.write(" ".join(names[self.encoded.ids[off[s]:off[s + 1]]]))
                fh.write("\n")


def _zipf_draws(rng: np.random.Generator, n: int, vocab_size: int, s: float,
                chunk: int = 1 << 24) -> np.ndarray:
    ranks = np.arange(1, vocab_size + 1, dtype=np.float64)
    cdf = np.cumsum(ranks ** (-s))
    cdf /= cdf[-1]
    out = np.empty(n, dtype=np.int32)
    for lo in range(0, n, chunk):
        hi = min(n, lo + chunk)
        u = rng.random(hi - lo)
        out[lo:hi] = np.minimum(np.searchsorted(cdf, u, side="right"), vocab_size - 1)
    return out


def _digits(x: np.ndarray) -> np.ndarray:
    d = np.ones_like(x, dtype=np.int64)
    v = x.astype(np.int64).copy()
    while True:
        v //= 10
        more = v > 0
        if not more.any():
            return d
        d += more


def make_planted_corpus(
    n_tokens: int,
    vocab_size: int,
    zipf_s: float = 1.0,
    n_clusters: int = 50,
    cluster_size: int = 20,
    sentence_len: int = 50,
    run_prob: float = 0.5,
    run_len: int = 8,
    min_count: int = 1,
    seed: int = 0,
) -> SyntheticCorpus:
    """Zipf(s) tokens over `vocab_size` raw ids with planted co-occurring clusters."""
    rng = np.random.default_rng(seed)
    raw = _zipf_draws(rng, n_tokens, vocab_size, zipf_s)
    n_sent = -(-n_tokens // sentence_len)
    # mid-frequency band: frequent enough to train, rare enough to survive t=1e-4
    need = n_clusters * cluster_size
    lo = max(1, vocab_size // 50)
    hi = max(lo + need, vocab_size // 5)
    hi = min(hi, vocab_size)
    if hi - lo < need:
        lo, hi = 0, vocab_size
    if need > vocab_size:
        raise ValueError("not enough ids for the requested clusters")
    members = rng.choice(np.arange(lo, hi), size=need, replace=False).astype(np.int32)
    raw_clusters = members.reshape(n_clusters, cluster_size)
    if n_clusters > 0 and run_len > 0:
        has_run = np.flatnonzero(rng.random(n_sent) < run_prob)
        which = rng.integers(0, n_clusters, size=len(has_run))
        for sent, c in zip(has_run, which):
            s_lo = int(sent) * sentence_len
            s_hi = min(n_tokens, s_lo + sentence_len)
            length = min(run_len, s_hi - s_lo)
            start = s_lo + int(rng.integers(0, s_hi - s_lo - length + 1))
            raw[start:start + length] = raw_clusters[c][rng.integers(0, cluster_size, size=length)]
    counts = np.bincount(raw, minlength=vocab_size).astype(np.int64)
    first = np.full(vocab_size, np.iinfo(np.int64).max, dtype=np.int64)
    _first_occurrence(raw, first)
    present = np.flatnonzero(counts >= max(1, min_count))
    order = present[np.lexsort((first[present], -counts[present]))]
    new_id = np.full(vocab_size, -1, dtype=np.int64)
    new_id[order] = np.arange(len(order))
    mapped = new_id[raw]
    keep = mapped >= 0
    sent_of = np.arange(n_tokens, dtype=np.int64) // sentence_len
    lens = np.bincount(sent_of[keep], minlength=n_sent)
    name_bytes = _digits(raw) + 2  # "w" + digits + separator
    sent_bytes = np.bincount(sent_of, weights=name_bytes, minlength=n_sent).astype(np.int64)
    nonempty = lens > 0
    offsets = np.concatenate([[0], np.cumsum(lens[nonempty])]).astype(np.int64)
    ids = mapped[keep].astype(np.int32)
    names = [f"w{r}" for r in order]
    vocab = Vocabulary(names, counts[order], {t: i for i, t in enumerate(names)},
                       int(counts[order].sum()))
    clusters = [new_id[c][new_id[c] >= 0] for c in raw_clusters]
    encoded = EncodedCorpus(ids, offsets, sent_bytes[nonempty])
    return SyntheticCorpus(vocab, encoded, clusters, seed)


def _first_occurrence(raw: np.ndarray, first: np.ndarray) -> None:
    # np.unique(return_index) gives the first index of each value
    vals, idx = np.unique(raw, return_index=True)
    first[vals] = idx


def tiny_config_corpus(seed: int = 0) -> SyntheticCorpus:
    """BASELINE.json configs[0]: 1M tokens, Zipf(1.0) over 10k ids, 50x20 clusters."""
    return make_planted_corpus(1_000_000, 10_000, zipf_s=1.0, seed=seed)


def mid_config_corpus(seed: int = 0) -> SyntheticCorpus:
    """BASELINE.json configs[2]: 17M tokens, Zipf(1.05) over 71k ids."""
    return make_planted_corpus(17_000_000, 71_000, zipf_s=1.05, seed=seed)


@dataclass
class DeviceSyntheticCorpus:
    """A planted-cluster corpus generated and kept in HBM (configs[3]: 800M tokens)."""

    ids: "object"            # torch int32 (device)
    offsets: "object"        # torch int64 (device)
    counts: np.ndarray       # int64 per final id (host)
    sentence_bytes: np.ndarray
    clusters: list[np.ndarray]
    n_tokens: int
    n_sentences: int
    max_sentence: int

    def vocabulary(self) -> Vocabulary:
        return Vocabulary.from_counts(self.counts)

    def host_offsets(self) -> np.ndarray:
        return self.offsets.cpu().numpy()

    def encoded(self, with_ids: bool = False) -> EncodedCorpus:
        ids = self.ids.cpu().numpy() if with_ids else np.empty(0, dtype=np.int32)
        return EncodedCorpus(ids, self.host_offsets(), self.sentence_bytes)


def make_planted_corpus_device(
    n_tokens: int,
    vocab_size: int,
    zipf_s: float = 1.05,
    n_clusters: int = 50,
    cluster_size: int = 20,
    sentence_len: int = 50,
    run_prob: float = 0.5,
    run_len: int = 8,
    min_count: int = 5,
    seed: int = 0,
    device: str = "cuda",
    chunk: int = 1 << 26,
) -> DeviceSyntheticCorpus:
    """Same construction as make_planted_corpus, generated with torch on the GPU
    (seeded torch Philox), so 800M-token corpora take seconds instead of minutes.
    Ids follow the reference vocabulary order (count desc, first occurrence);
    ids with count < min_count are dropped as encode_corpus drops OOV tokens."""
    import torch

    g = torch.Generator(device=device)
    g.manual_seed(seed)
    V = vocab_size
    ranks = torch.arange(1, V + 1, dtype=torch.float64, device=device)
    cdf = torch.cumsum(ranks.pow(-zipf_s), 0)
    cdf /= cdf[-1].clone()
    raw = torch.empty(n_tokens, dtype=torch.int32, device=device)
    for lo in range(0, n_tokens, chunk):
        hi = min(n_tokens, lo + chunk)
        u = torch.rand(hi - lo, generator=g, dtype=torch.float64, device=device)
        raw[lo:hi] = torch.searchsorted(cdf, u, right=True).clamp_(max=V - 1).to(torch.int32)
        del u
    rng = np.random.default_rng(seed)
    need = n_clusters * cluster_size
    band_lo = max(1, V // 50)
    band_hi = min(max(band_lo + need, V // 5), V)
    if band_hi - band_lo < need:
        band_lo, band_hi = 0, V
    members = rng.choice(np.arange(band_lo, band_hi), size=need, replace=False).astype(np.int32)
    raw_clusters = members.reshape(n_clusters, cluster_size)
    n_sent = -(-n_tokens // sentence_len)
    if n_clusters > 0 and run_len > 0:
        sel = torch.nonzero(torch.rand(n_sent, generator=g, device=device) < run_prob).flatten()
        ns = sel.numel()
        s_lo = sel * sentence_len
        s_len = torch.clamp(n_tokens - s_lo, max=sentence_len)
        length = torch.clamp(s_len, max=run_len)
        start = s_lo + (torch.rand(ns, generator=g, device=device) * (s_len - length + 1)).long()
        cl = torch.randint(0, n_clusters, (ns,), generator=g, device=device)
        dev_members = torch.from_numpy(raw_clusters).to(device)
        for j in range(run_len):
            ok = j < length
            pos = (start + j)[ok]
            pick = torch.randint(0, cluster_size, (ns,), generator=g, device=device)[ok]
            raw[pos] = dev_members[cl[ok], pick]
    counts = torch.bincount(raw, minlength=V)
    first = torch.full((V,), n_tokens, dtype=torch.int64, device=device)
    for lo in range(0, n_tokens, chunk):
        hi = min(n_tokens, lo + chunk)
        first.scatter_reduce_(0, raw[lo:hi].long(),
                              torch.arange(lo, hi, dtype=torch.int64, device=device), "amin")
    present = counts >= max(1, min_count)
    key = torch.where(present, (-counts) * (n_tokens + 1) + first,
                      torch.full_like(first, torch.iinfo(torch.int64).max))
    n_present = int(present.sum().item())
    order = torch.argsort(key)[:n_present]
    new_id = torch.full((V,), -1, dtype=torch.int32, device=device)
    new_id[order] = torch.arange(n_present, dtype=torch.int32, device=device)
    lens = torch.zeros(n_sent, dtype=torch.int64, device=device)
    sbytes = torch.zeros(n_sent, dtype=torch.float64, device=device)
    digits = torch.floor(torch.log10(torch.arange(V, device=device, dtype=torch.float64).clamp(min=1))) + 3
    pieces = []
    for lo in range(0, n_tokens, chunk):
        hi = min(n_tokens, lo + chunk)
        r = raw[lo:hi].long()
        mapped = new_id[r]
        keep = mapped >= 0
        sent = torch.arange(lo, hi, dtype=torch.int64, device=device) // sentence_len
        lens += torch.bincount(sent[keep], minlength=n_sent)
        sbytes += torch.bincount(sent, weights=digits[r], minlength=n_sent)
        pieces.append(mapped[keep])
        del r, mapped, keep, sent
    del raw, first
    ids = torch.cat(pieces)
    del pieces
    nonempty = lens > 0
    lens_ne = lens[nonempty]
    offsets = torch.zeros(int(lens_ne.numel()) + 1, dtype=torch.int64, device=device)
    offsets[1:] = torch.cumsum(lens_ne, 0)
    counts_host = counts[order].cpu().numpy().astype(np.int64)
    new_host = new_id.cpu().numpy()
    clusters = [new_host[c][new_host[c] >= 0].astype(np.int64) for c in raw_clusters]
    return DeviceSyntheticCorpus(ids, offsets, counts_host,
                                 sbytes[nonempty].cpu().numpy().astype(np.int64), clusters,
                                 int(ids.numel()), int(lens_ne.numel()),
                                 int(lens_ne.max().item()) if lens_ne.numel() else 0)


def large_config_corpus(seed: int = 0, n_tokens: int = 800_000_000, device: str = "cuda"):
    """BASELINE.json configs[3]: 800M tokens, Zipf(1.05) over 1M ids, min-count 5."""
    return make_planted_corpus_device(n_tokens, 1_000_000, zipf_s=1.05, min_count=5, seed=seed,
                                      device=device)
