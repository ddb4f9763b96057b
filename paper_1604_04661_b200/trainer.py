"""Training entry points over the device driver (drop-in for sgns/trainer.py).

Reference map:
  ALPHA_REFRESH_WORDS          sgns/trainer.py:48
  ConfigError / TrainingConfig sgns/trainer.py:51-109
  TrainingStats                sgns/trainer.py:112-119
  update_alpha                 sgns/trainer.py:122-132
  ThreadRun.advance            sgns/trainer.py:396-453  -> DeviceRun.advance (all workers, one launch)
  train_encoded / train        sgns/trainer.py:477-552

A reference thread is a device worker (one warp): it owns a contiguous
sentence range from `split_by_tokens`, keeps its own stream and counters, and
shares the model without locks (Hogwild).  Two samplers:
  rng="splitmix"  the reference's per-thread splitmix64 stream (seed, stream
                  id) and its count^0.75 slot table; with workers == threads
                  every window, chunk and negative is bit-identical to the
                  reference's, and alpha refreshes every 10,000 words per worker.
  rng="philox"    production: Philox4x32-10 keyed by seed, counter = corpus
                  token position (partition-invariant) and an alias table;
                  alpha refreshes every sentence from the shared words-read
                  counter, so it tracks global progress with ~1500 workers.
"""

from __future__ import annotations

import time
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .corpus import (KEPT_BUFFER_TOKENS, EncodedCorpus, NegativeTable, Vocabulary, build_vocab,
                     default_table_length, encode_corpus, negative_table_boundaries,
                     read_tokens, split_by_tokens, NEGATIVE_POWER)
from .model import DeviceModel, EmbeddingModel, current_stream_ptr, init_device_model, padded_ld
from .kernel_batched import device_sigmoid_table
from .rng import new_state

ALPHA_REFRESH_WORDS = 10_000
_INF_BUDGET = 2**62

WORKER_DTYPE = np.dtype([
    ("next_sent", "<i8"), ("lo", "<i8"), ("hi", "<i8"), ("epoch", "<i4"), ("done", "<i4"),
    ("rng", "<u8"), ("alpha", "<f8"), ("read_local", "<f8"), ("trained_local", "<f8"),
    ("kernel_counter", "<i8"), ("words_read", "<i8"), ("words_trained", "<i8"), ("inputs", "<i8")])


DEVICE_ERRORS = {
    1: "a window with no inputs or more inputs than the staging holds",
    2: "sentence longer than the kept-token buffer",
    3: "negative sampling drew 2^17 candidates without finding K words different from the "
       "target (the target holds almost all of the count^0.75 mass)",
}


class ConfigError(ValueError):
    """Invalid training configuration."""


@dataclass
class TrainingConfig:
    dim: int = 300
    window: int = 5
    negatives: int = 5
    subsample: float = 1e-4
    min_count: int = 5
    alpha0: float = 0.025
    alpha_floor_fraction: float = 1e-4
    epochs: int = 5
    threads: int = 1
    batch_cap: int = 16
    kernel: str = "batched"
    seed: int = 1
    dynamic_window: bool = True
    table_length: int | None = None
    float64: bool = False
    matmul: str | None = None  # None / "cuda" / the reference's "blas" | "naive" (all the CUDA core)
    loss_sample_every: int = 100
    # device knobs (new)
    rng: str = "philox"                   # "philox" (production) | "splitmix" (reference stream)
    workers: int | None = None            # None: splitmix -> threads; philox -> resident warps
    alpha_refresh_words: int | None = None  # None: splitmix -> 10,000; philox -> every sentence
    schedule: str = "auto"                # "auto" | "static" (fixed ranges) | "dynamic" (claims)

    def validate(self) -> None:
        if self.dim < 1:
            raise ConfigError("dim must be >= 1")
        if self.window < 1:
            raise ConfigError("window must be >= 1")
        if self.negatives < 1:
            raise ConfigError("negatives must be >= 1")
        if self.negatives > 31:
            raise ConfigError("negatives must be <= 31 on the device path")
        if self.subsample < 0:
            raise ConfigError("subsample must be >= 0")
        if self.min_count < 1:
            raise ConfigError("min_count must be >= 1")
        if self.alpha0 <= 0:
            raise ConfigError("alpha0 must be positive")
        if not 0 < self.alpha_floor_fraction < 1:
            raise ConfigError("alpha_floor_fraction must be in (0, 1)")
        if self.epochs < 1:
            raise ConfigError("epochs must be >= 1")
        if self.threads < 1:
            raise ConfigError("threads must be >= 1")
        if self.batch_cap < 1:
            raise ConfigError("batch_cap must be >= 1")
        if self.kernel != "batched":
            raise ConfigError(f"unknown kernel {self.kernel!r} (the device path is 'batched')")
        if self.matmul not in (None, "cuda", "blas", "naive"):
            raise ConfigError(f"unknown matmul backend {self.matmul!r}")
        if self.rng not in ("philox", "splitmix"):
            raise ConfigError(f"unknown rng {self.rng!r}")
        if self.workers is not None and self.workers < 1:
            raise ConfigError("workers must be >= 1")
        if self.alpha_refresh_words is not None and self.alpha_refresh_words < 1:
            raise ConfigError("alpha_refresh_words must be >= 1")
        if self.schedule not in ("auto", "static", "dynamic"):
            raise ConfigError(f"unknown schedule {self.schedule!r}")
        if self.rng == "philox" and -(-2 * self.window // self.batch_cap) > 256:
            # the Philox negative counter keeps 8 bits of the chunk index (csrc/sgns_device.cuh)
            raise ConfigError("rng='philox' supports at most 256 chunks per position "
                              "(ceil(2 * window / batch_cap) <= 256)")
        if self.schedule == "dynamic" and not self.dynamic_eligible(0):
            raise ConfigError("schedule='dynamic' needs rng='philox', float32, negatives <= 15, dim <= 512")

    def dynamic_eligible(self, vocab_size: int) -> bool:
        cols = -(-self.dim // 4) * 4
        ld = padded_ld(self.dim, np.float32)
        return (self.rng == "philox" and not self.float64 and self.negatives + 1 <= 16
                and -(-(cols // 2) // 32) <= 8 and vocab_size * ld < 2**32)

    def use_dynamic(self, vocab_size: int) -> bool:
        if self.schedule == "static":
            return False
        return self.dynamic_eligible(vocab_size)

    @property
    def dtype(self):
        return np.float64 if self.float64 else np.float32

    @property
    def refresh_words(self) -> int:
        if self.alpha_refresh_words is not None:
            return self.alpha_refresh_words
        return ALPHA_REFRESH_WORDS if self.rng == "splitmix" else 1


@dataclass
class TrainingStats:
    words_processed: int = 0
    words_read: int = 0
    wall_seconds: float = 0.0
    throughput_words_per_sec: float = 0.0
    final_alpha: float = 0.0
    loss_by_epoch: list[float] = field(default_factory=list)


def update_alpha(words_done: int, total_words_times_epochs: float, alpha0: float,
                 floor_fraction: float) -> float:
    frac = 1.0 - words_done / (total_words_times_epochs + 1.0)
    if frac < floor_fraction:
        frac = floor_fraction
    return alpha0 * frac


def _torch():
    import torch
    if not torch.cuda.is_available():
        raise RuntimeError("paper_1604_04661_b200 needs a CUDA device (no CPU fallback)")
    return torch


class DeviceCorpus:
    """EncodedCorpus resident in HBM (int32 ids, int64 sentence offsets)."""

    def __init__(self, encoded: EncodedCorpus, device="cuda", ids=None, offsets=None):
        torch = _torch()
        self.host_offsets = np.ascontiguousarray(encoded.offsets, dtype=np.int64)
        self.n_sentences = encoded.n_sentences
        self.n_tokens = encoded.n_tokens
        self.max_sentence = encoded.max_sentence_length()
        if self.max_sentence > KEPT_BUFFER_TOKENS:
            raise ValueError(f"sentence of {self.max_sentence} tokens exceeds the device limit "
                             f"{KEPT_BUFFER_TOKENS} (encode_corpus splits at 1000)")
        self.ids = ids if ids is not None else torch.from_numpy(
            np.ascontiguousarray(encoded.ids, dtype=np.int32)).to(device)
        self.offsets = offsets if offsets is not None else torch.from_numpy(self.host_offsets).to(device)
        if self.ids.numel() < self.n_tokens:
            raise ValueError("corpus ids shorter than its offsets")
        if self.n_tokens:
            lo, hi = torch.aminmax(self.ids[:self.n_tokens])
            self.id_range = (int(lo.item()), int(hi.item()))
        else:
            self.id_range = (0, -1)

    def check_vocab(self, vocab_size: int) -> None:
        """The kernels do not bounds-check ids (as the reference's numba cores); refuse here."""
        if self.id_range[0] < 0 or self.id_range[1] >= vocab_size:
            raise ValueError(f"corpus ids span {self.id_range}, outside a vocabulary of {vocab_size}")


class DeviceSampler:
    """Negative sampler in HBM: the reference slot table or the alias table."""

    def __init__(self, counts: np.ndarray, rng: str, table_length: int | None = None,
                 table: NegativeTable | None = None, device="cuda", power: float = NEGATIVE_POWER):
        self.rng = rng
        counts = np.ascontiguousarray(counts, dtype=np.int64)
        V = len(counts)
        self.vocab = V
        self.slots = self.alias_thr = self.alias_idx = None
        if rng == "splitmix":
            if table is not None:
                bounds = np.ascontiguousarray(table.boundaries, dtype=np.int64)
            else:
                L = table_length if table_length is not None else default_table_length(V)
                if L < V:
                    from .corpus import TableLengthError
                    raise TableLengthError(f"table length {L} is smaller than vocabulary size {V}")
                bounds = negative_table_boundaries(counts, power, L)
            if np.count_nonzero(np.diff(bounds, prepend=0)) < 2:
                raise ValueError("negative table holds fewer than two distinct words: every draw "
                                 "would equal the target (the reference's rejection loop never ends)")
        elif np.count_nonzero(counts > 0) < 2:
            raise ValueError("fewer than two words with a positive count: no negative can "
                             "differ from the target")
        torch = _torch()
        if rng == "splitmix":
            n = int(bounds[-1])
            d_bounds = torch.from_numpy(bounds).to(device)
            self.slots = torch.empty(n, dtype=torch.int32, device=device)
            rc = _lib.lib().sgns_expand_slots(d_bounds.data_ptr(), V, self.slots.data_ptr(), n,
                                              current_stream_ptr(d_bounds.device))
            _lib.check(rc, "sgns_expand_slots")
        else:
            thr = np.empty(V, dtype=np.uint32)
            idx = np.empty(V, dtype=np.int32)
            rc = _lib.lib().sgns_build_alias(counts.ctypes.data, V, power, thr.ctypes.data,
                                             idx.ctypes.data)
            _lib.check(rc, "sgns_build_alias")
            self.host_alias = (thr, idx)
            self.alias_thr = torch.from_numpy(thr.view(np.int32)).to(device)
            self.alias_idx = torch.from_numpy(idx).to(device)


def resident_workers(config: TrainingConfig, max_sentence: int) -> int:
    out = _lib.I32(0)
    rc = _lib.lib().sgns_resident_workers(
        _lib.SGNS_F64 if config.float64 else _lib.SGNS_F32, config.dim, config.window,
        config.negatives, config.batch_cap, max(max_sentence, 1), out)
    _lib.check(rc, "sgns_resident_workers")
    return int(out.value)


class DeviceRun:
    """All device workers of one rank: ThreadRun (trainer.py:332-453) x W, one launch per advance."""

    def __init__(self, model: DeviceModel, corpus: DeviceCorpus, sampler: DeviceSampler,
                 keep_probs: np.ndarray | None, config: TrainingConfig, alpha0_eff: float,
                 total_x_epochs: float, n_workers: int, sent_range: tuple[int, int] | None = None,
                 stream_base: int = 0, trace_cap: int = 0, update: bool = True,
                 track_dirty: bool = False):
        torch = _torch()
        self.torch = torch
        corpus.check_vocab(model.vocab_size)
        if sampler.vocab != model.vocab_size:
            raise ValueError("sampler and model vocabulary sizes differ")
        self.model, self.corpus, self.sampler, self.config = model, corpus, sampler, config
        dev = model.m_in.device
        self.device = dev
        lo, hi = sent_range if sent_range is not None else (0, corpus.n_sentences)
        ranges = split_by_tokens(corpus.host_offsets, lo, hi, n_workers)
        w = np.zeros(n_workers, dtype=WORKER_DTYPE)
        w["lo"] = [a for a, _ in ranges]
        w["next_sent"] = w["lo"]
        w["hi"] = [b for _, b in ranges]
        w["alpha"] = alpha0_eff
        if config.rng == "splitmix":
            w["rng"] = [new_state(config.seed, stream_base + i) for i in range(n_workers)]
        self.n_workers = n_workers
        self.workers = torch.from_numpy(w.view(np.uint8)).to(dev)
        self.shared = torch.zeros(2, dtype=torch.int64, device=dev)
        self.loss = torch.zeros((n_workers, config.epochs), dtype=torch.float64, device=dev)
        self.cells = torch.zeros((n_workers, config.epochs), dtype=torch.int64, device=dev)
        self.error = torch.zeros(1, dtype=torch.int32, device=dev)
        self.keep = None if keep_probs is None else torch.from_numpy(
            np.ascontiguousarray(keep_probs, dtype=np.float64)).to(dev)
        self.sig = device_sigmoid_table(model.np_dtype, dev)
        k1 = config.negatives + 1
        self.rec_len = 4 + config.batch_cap + k1
        self.trace_cap = trace_cap
        if trace_cap:
            self.trace = torch.full((n_workers, trace_cap, self.rec_len), -1, dtype=torch.int32, device=dev)
            self.trace_alpha = torch.zeros((n_workers, trace_cap), dtype=torch.float64, device=dev)
            self.trace_count = torch.zeros(n_workers, dtype=torch.int64, device=dev)
        self.alpha0_eff = alpha0_eff
        self.total_x_epochs = total_x_epochs
        p = _lib.DriveParams()
        p.dtype = model.cdtype
        p.d_m_in, p.d_m_out = model.m_in.data_ptr(), model.m_out.data_ptr()
        p.vocab, p.ld, p.dim = model.vocab_size, model.ld, model.dim
        p.d_ids, p.d_offsets = corpus.ids.data_ptr(), corpus.offsets.data_ptr()
        p.d_keep_probs = None if self.keep is None else self.keep.data_ptr()
        p.rng_mode = _lib.RNG_SPLITMIX if config.rng == "splitmix" else _lib.RNG_PHILOX
        if sampler.slots is not None:
            p.d_slots, p.n_slots = sampler.slots.data_ptr(), sampler.slots.numel()
        if sampler.alias_thr is not None:
            p.d_alias_thr, p.d_alias_idx = sampler.alias_thr.data_ptr(), sampler.alias_idx.data_ptr()
        p.seed = config.seed & (2**64 - 1)
        p.window, p.dynamic, p.k_neg = config.window, int(config.dynamic_window), config.negatives
        p.batch_cap = config.batch_cap
        p.sigmoid_mode = _lib.SIGMOID_EXACT if config.float64 else _lib.SIGMOID_TABLE
        p.d_sig_table = self.sig.data_ptr()
        p.alpha0, p.floor_frac = alpha0_eff, config.alpha_floor_fraction
        p.total_x_epochs = total_x_epochs
        p.refresh_words = config.refresh_words
        p.d_shared = self.shared.data_ptr()
        p.epochs, p.loss_every = config.epochs, config.loss_sample_every
        p.d_workers, p.n_workers = self.workers.data_ptr(), n_workers
        p.d_loss_by_epoch, p.d_cells_by_epoch = self.loss.data_ptr(), self.cells.data_ptr()
        p.update = int(update)
        p.max_sentence = max(corpus.max_sentence, 1)
        if trace_cap:
            p.trace_cap = trace_cap
            p.d_trace, p.d_trace_alpha = self.trace.data_ptr(), self.trace_alpha.data_ptr()
            p.d_trace_count = self.trace_count.data_ptr()
        p.d_error = self.error.data_ptr()
        # touched-row map (M_in rows, M_out rows) for data-parallel touched-row averaging
        self.dirty = None
        if track_dirty:
            self.dirty = torch.zeros((2, model.vocab_size), dtype=torch.uint8, device=dev)
            p.d_dirty = self.dirty.data_ptr()
        self.dynamic = config.use_dynamic(model.vocab_size)
        if self.dynamic:
            # sentence ordinals c in [0, epochs * n) of the shard, claimed by the workers
            self.shard_lo, self.shard_hi = lo, hi
            self.n_sent = hi - lo
            offs = corpus.host_offsets
            self._offs = offs
            self.shard_tokens = int(offs[hi] - offs[lo])
            self.total_claims = config.epochs * self.n_sent
            self.claim_pos = 0
            self.claim = torch.zeros(1, dtype=torch.int64, device=dev)
            p.schedule = _lib.SCHEDULE_DYNAMIC
            p.d_claim = self.claim.data_ptr()
            p.shard_lo, p.shard_hi = lo, hi
            self._dyn_read = 0
            if trace_cap:
                self.trace = torch.full((trace_cap, self.rec_len), -1, dtype=torch.int32, device=dev)
                self.trace_alpha = torch.zeros(trace_cap, dtype=torch.float64, device=dev)
                self.trace_count = torch.zeros(1, dtype=torch.int64, device=dev)
                p.d_trace, p.d_trace_alpha = self.trace.data_ptr(), self.trace_alpha.data_ptr()
                p.d_trace_count = self.trace_count.data_ptr()
        self.params = p
        self._host_state = None

    # -- dynamic schedule helpers -------------------------------------------
    def words_at(self, c: int) -> int:
        """Words read by this shard before sentence ordinal c (epoch-major)."""
        if self.n_sent == 0:
            return 0
        e, r = divmod(int(c), self.n_sent)
        return e * self.shard_tokens + int(self._offs[self.shard_lo + r] - self._offs[self.shard_lo])

    def _claim_end(self, budget_total: int) -> int:
        start = self.claim_pos
        target = self.words_at(start) + budget_total
        lo, hi = start + 1, self.total_claims
        if lo > hi:
            return hi
        if self.words_at(hi) < target:
            return hi
        while lo < hi:  # smallest c with words_at(c) >= target
            mid = (lo + hi) // 2
            if self.words_at(mid) >= target:
                hi = mid
            else:
                lo = mid + 1
        return lo

    # -- launches ---------------------------------------------------------
    def launch(self, word_budget: int, stream=None) -> None:
        """Stream-ordered: every worker consumes up to word_budget words read
        (dynamic schedule: the workers together consume n_workers * word_budget)."""
        self.params.word_budget = int(word_budget)
        st = current_stream_ptr(self.device) if stream is None else stream
        if self.dynamic:
            if self.claim_pos >= self.total_claims:
                return
            total = min(int(word_budget) * self.n_workers, 2**62)
            end = self._claim_end(total)
            if stream is None:
                self.claim.fill_(self.claim_pos)
            else:  # the claim counter is reset on the launch's own stream
                with self.torch.cuda.stream(self.torch.cuda.ExternalStream(st, device=self.device)):
                    self.claim.fill_(self.claim_pos)
            self.params.claim_end = end
            self._dyn_read += self.words_at(end) - self.words_at(self.claim_pos)
            self.claim_pos = end
        _lib.check(_lib.lib().sgns_drive(self.params, st), "sgns_drive")
        self._host_state = None

    def state(self) -> np.ndarray:
        if self._host_state is None:
            self._host_state = self.workers.cpu().numpy().view(WORKER_DTYPE).copy()
            err = int(self.error.item())
            if err:
                raise RuntimeError(f"sgns_drive device error {err}: {DEVICE_ERRORS.get(err, 'unknown')}")
        return self._host_state

    @property
    def done(self) -> bool:
        if self.dynamic:
            return self.claim_pos >= self.total_claims
        return bool(self.state()["done"].all())

    @property
    def words_read(self) -> int:
        if self.dynamic:
            return self._dyn_read
        return int(self.state()["words_read"].sum())

    @property
    def words_trained(self) -> int:
        return int(self.state()["words_trained"].sum())

    def advance(self, word_budget: int) -> int:
        """ThreadRun.advance semantics per worker; returns words read by all workers."""
        before = self.words_read
        self.launch(word_budget)
        return self.words_read - before

    def run_to_completion(self) -> None:
        while not self.done:
            self.launch(_INF_BUDGET // max(self.n_workers, 1))

    def loss_by_epoch(self) -> list[float]:
        ls = self.loss.sum(dim=0).cpu().numpy()
        cs = self.cells.sum(dim=0).cpu().numpy()
        return [float(a / b) if b else 0.0 for a, b in zip(ls, cs)]

    def shared_words_read(self) -> int:
        if self.dynamic:
            return self.words_at(self.claim_pos)
        return int(self.shared[0].item())

    def trace_records(self):
        """Dynamic schedule: every traced window (processing order across workers)."""
        n = min(int(self.trace_count[0].item()), self.trace_cap)
        return self.trace[:n].cpu().numpy(), self.trace_alpha[:n].cpu().numpy()

    def worker_trace(self, w: int):
        n = min(int(self.trace_count[w].item()), self.trace_cap)
        return self.trace[w, :n].cpu().numpy(), self.trace_alpha[w, :n].cpu().numpy()


MIN_TOKENS_PER_WORKER = 2048


def default_workers(config: TrainingConfig, corpus: DeviceCorpus, n_sentences: int | None = None,
                    n_tokens: int | None = None) -> int:
    """Workers in flight: every resident warp, but at most one per 2,048 corpus tokens,
    which bounds Hogwild staleness on small corpora (+0.3% loss at 512
    workers, +1.2% at 2,048 on a 10k vocabulary); large corpora use the whole GPU."""
    if config.workers is not None:
        return config.workers
    if config.rng == "splitmix":
        return config.threads
    cap = resident_workers(config, corpus.max_sentence)
    n = corpus.n_sentences if n_sentences is None else n_sentences
    toks = corpus.n_tokens if n_tokens is None else n_tokens
    return max(1, min(cap, n, toks // MIN_TOKENS_PER_WORKER))


def train_encoded(vocab: Vocabulary, encoded: EncodedCorpus, config: TrainingConfig,
                  model: EmbeddingModel | DeviceModel | None = None,
                  table: NegativeTable | None = None, progress: bool = False,
                  return_device: bool = False):
    """Train over an encoded corpus on the GPU; returns (model, TrainingStats)."""
    config.validate()
    torch = _torch()
    if model is None:
        dm = init_device_model(vocab.size, config.dim, config.seed, config.dtype)
    elif isinstance(model, DeviceModel):
        dm = model
    else:
        dm = DeviceModel.from_host(model)
    corpus = DeviceCorpus(encoded, dm.m_in.device)
    sampler = DeviceSampler(vocab.counts, config.rng, config.table_length, table, dm.m_in.device)
    keep = vocab.keep_probs(config.subsample) if config.subsample > 0 else None
    total_x_epochs = float(encoded.n_tokens) * config.epochs
    n_workers = default_workers(config, corpus)
    run = DeviceRun(dm, corpus, sampler, keep, config, config.alpha0, total_x_epochs, n_workers)
    torch.cuda.synchronize(dm.m_in.device)
    started = time.perf_counter()
    run.run_to_completion()
    torch.cuda.synchronize(dm.m_in.device)
    wall = time.perf_counter() - started
    stats = TrainingStats()
    stats.words_processed = run.words_trained
    stats.words_read = run.words_read
    stats.wall_seconds = wall
    stats.throughput_words_per_sec = stats.words_processed / max(wall, 1e-9)
    stats.final_alpha = update_alpha(run.shared_words_read(), total_x_epochs, config.alpha0,
                                     config.alpha_floor_fraction)
    stats.loss_by_epoch = run.loss_by_epoch()
    if return_device:
        return dm, stats
    if isinstance(model, EmbeddingModel):
        dm.copy_to_host(model)
        return model, stats
    return dm.to_host(), stats


def train(corpus_path: str, config: TrainingConfig, progress: bool = False):
    """Build the vocabulary, encode the corpus (multithreaded C++ scanner, identical to
    build_vocab/encode_corpus), and train a fresh model on the GPU."""
    from .corpus import build_vocab_file, encode_corpus_file
    config.validate()
    vocab = build_vocab_file(corpus_path, config.min_count)
    encoded = encode_corpus_file(corpus_path, vocab)
    model, stats = train_encoded(vocab, encoded, config, progress=progress)
    return model, vocab, stats


class StreamingTrainer:
    """Out-of-core training: sentence chunks stream from pinned host memory through
    two preallocated HBM buffer sets while the model, sampler and alpha schedule stay
    resident.  `train_chunks` pipelines: chunk i+1's host->device copy runs on a side
    stream while chunk i trains, and chunk i's counters (accumulated by the kernel into
    a 64-byte totals block) are read back once chunk i+1 is launched.  Draws are keyed
    by the global corpus position (`token_base`) and alpha by the global words-read
    position, so chunking does not change the training."""

    def __init__(self, model: DeviceModel, counts: np.ndarray, config: TrainingConfig,
                 total_x_epochs: float, max_chunk_tokens: int, max_chunk_sentences: int,
                 max_sentence: int, n_workers: int | None = None, alpha0_eff: float | None = None,
                 keep_probs: np.ndarray | None = None):
        torch = _torch()
        config.validate()
        if not config.use_dynamic(model.vocab_size):
            raise ConfigError("streaming training needs the dynamic schedule "
                              "(rng='philox', float32, negatives <= 15, dim <= 512)")
        self.torch = torch
        self.model, self.config = model, config
        dev = model.m_in.device
        self.device = dev
        self.max_tok, self.max_sent = max_chunk_tokens, max_chunk_sentences
        self.ids = [torch.empty(max_chunk_tokens, dtype=torch.int32, device=dev) for _ in range(2)]
        self.offsets = [torch.empty(max_chunk_sentences + 1, dtype=torch.int64, device=dev) for _ in range(2)]
        self.off_pinned = [torch.empty(max_chunk_sentences + 1, dtype=torch.int64).pin_memory()
                           for _ in range(2)]
        self.acc = [torch.zeros(8, dtype=torch.int64, device=dev) for _ in range(2)]  # totals + loss
        self.acc_host = [torch.zeros(8, dtype=torch.int64).pin_memory() for _ in range(2)]
        self.copy_stream = torch.cuda.Stream(dev)
        self.copied = [torch.cuda.Event() for _ in range(2)]
        self.trained_ev = [torch.cuda.Event() for _ in range(2)]
        self.read_ev = [torch.cuda.Event() for _ in range(2)]
        self.sampler = DeviceSampler(counts, "philox", device=dev)
        if keep_probs is None and config.subsample > 0:
            from .corpus import keep_probabilities
            keep_probs = keep_probabilities(counts, int(np.sum(counts)), config.subsample)
        self.keep = None if keep_probs is None else torch.from_numpy(
            np.ascontiguousarray(keep_probs, dtype=np.float64)).to(dev)
        if n_workers is None:
            n_workers = resident_workers(config, max_sentence)
        self.n_workers = n_workers
        self.alpha0_eff = config.alpha0 if alpha0_eff is None else alpha0_eff
        self.total_x_epochs = total_x_epochs
        self.workers = torch.zeros((n_workers * WORKER_DTYPE.itemsize,), dtype=torch.uint8, device=dev)
        self.claim = torch.zeros(1, dtype=torch.int64, device=dev)
        self.loss = torch.zeros((n_workers, 1), dtype=torch.float64, device=dev)
        self.cells = torch.zeros((n_workers, 1), dtype=torch.int64, device=dev)
        self.shared = torch.zeros(2, dtype=torch.int64, device=dev)
        self.sig = device_sigmoid_table(model.np_dtype, dev)
        p = _lib.DriveParams()
        p.dtype = model.cdtype
        p.d_m_in, p.d_m_out = model.m_in.data_ptr(), model.m_out.data_ptr()
        p.vocab, p.ld, p.dim = model.vocab_size, model.ld, model.dim
        p.d_keep_probs = None if self.keep is None else self.keep.data_ptr()
        p.rng_mode = _lib.RNG_PHILOX
        p.d_alias_thr, p.d_alias_idx = self.sampler.alias_thr.data_ptr(), self.sampler.alias_idx.data_ptr()
        p.seed = config.seed & (2**64 - 1)
        p.window, p.dynamic, p.k_neg = config.window, int(config.dynamic_window), config.negatives
        p.batch_cap = config.batch_cap
        p.sigmoid_mode = _lib.SIGMOID_TABLE
        p.d_sig_table = self.sig.data_ptr()
        p.alpha0, p.floor_frac = self.alpha0_eff, config.alpha_floor_fraction
        p.total_x_epochs = total_x_epochs
        p.refresh_words = config.refresh_words
        p.d_shared = self.shared.data_ptr()
        p.epochs, p.loss_every = 1, config.loss_sample_every
        p.d_workers, p.n_workers = self.workers.data_ptr(), n_workers
        p.d_loss_by_epoch, p.d_cells_by_epoch = self.loss.data_ptr(), self.cells.data_ptr()
        p.update = 1
        p.max_sentence = max(max_sentence, 1)
        p.word_budget = _INF_BUDGET
        p.schedule = _lib.SCHEDULE_DYNAMIC
        p.d_claim = self.claim.data_ptr()
        p.shard_lo = 0
        self.params = p
        self.h2d_bytes = 0
        self.d2h_bytes = 0

    def _stage(self, buf: int, ids_host, offsets_host) -> tuple[int, int]:
        """Queue the host->device copies of one chunk into buffer set `buf` (side stream)."""
        torch = self.torch
        n_sent = len(offsets_host) - 1
        n_tok = int(offsets_host[-1])
        if n_tok > self.max_tok or n_sent > self.max_sent:
            raise ValueError("chunk larger than the streaming buffers")
        if torch.is_tensor(offsets_host) and offsets_host.is_pinned():
            off_src = offsets_host
        else:
            self.copied[buf].synchronize()  # the staging buffer's previous copy has landed
            self.off_pinned[buf][:n_sent + 1].copy_(torch.as_tensor(np.asarray(offsets_host, dtype=np.int64)))
            off_src = self.off_pinned[buf][:n_sent + 1]
        with torch.cuda.stream(self.copy_stream):
            self.copy_stream.wait_event(self.trained_ev[buf])  # previous user of this buffer set
            self.ids[buf][:n_tok].copy_(ids_host[:n_tok], non_blocking=True)
            self.offsets[buf][:n_sent + 1].copy_(off_src, non_blocking=True)
            self.copied[buf].record(self.copy_stream)
        return n_tok, n_sent

    def _launch(self, buf: int, n_tok: int, n_sent: int, token_base: int, epoch: int, words_base: int):
        torch = self.torch
        stream = torch.cuda.current_stream(self.device)
        stream.wait_event(self.copied[buf])
        self.acc[buf].zero_()
        p = self.params
        p.d_ids, p.d_offsets = self.ids[buf].data_ptr(), self.offsets[buf].data_ptr()
        p.shard_hi = n_sent
        p.claim_end = n_sent
        p.token_base = int(token_base)
        p.epoch_base = int(epoch)
        p.words_base = int(words_base)
        p.d_totals = self.acc[buf].data_ptr()
        p.d_loss_total = self.acc[buf][6:7].data_ptr()
        self.claim.zero_()
        _lib.check(_lib.lib().sgns_drive(p, stream.cuda_stream), "sgns_drive")
        self.trained_ev[buf].record(stream)
        self.acc_host[buf].copy_(self.acc[buf], non_blocking=True)
        self.read_ev[buf].record(stream)
        self.h2d_bytes = n_tok * 4 + (n_sent + 1) * 8
        self.d2h_bytes = self.acc_host[buf].numel() * 8

    def _result(self, buf: int):
        self.read_ev[buf].synchronize()
        a = self.acc_host[buf].numpy()
        loss = float(a[6:7].view(np.float64)[0])
        # (words_trained, words_read, loss_sum, loss_cells, inputs, chunks)
        return int(a[0]), int(a[1]), loss, int(a[4]), int(a[3]), int(a[2])

    def train_chunks(self, chunks, after_launch=None):
        """Train an iterable of (ids_host, offsets_host, token_base[, epoch[, words_base]])
        chunks with copy/compute overlap; yields each chunk's counters in order.
        `after_launch()`, if given, runs after each chunk's kernel is enqueued and before
        the next one is: stream-ordered work between chunks (the data-parallel model
        average, sgns/distributed.py:470-472)."""
        it = iter(chunks)
        try:
            nxt = next(it)
        except StopIteration:
            return
        buf = 0
        staged = self._stage(buf, nxt[0], nxt[1])
        pending = None
        while nxt is not None:
            cur, cur_buf, cur_staged = nxt, buf, staged
            try:
                nxt = next(it)
            except StopIteration:
                nxt = None
            if cur_staged[1] > 0:
                epoch = cur[3] if len(cur) > 3 else 0
                words_base = cur[4] if len(cur) > 4 else cur[2]
                self._launch(cur_buf, cur_staged[0], cur_staged[1], cur[2], epoch, words_base)
            if after_launch is not None:
                after_launch()
            if nxt is not None:
                buf ^= 1
                staged = self._stage(buf, nxt[0], nxt[1])
            if pending is not None:
                yield self._result(pending) if pending >= 0 else (0, 0, 0.0, 0, 0, 0)
            pending = cur_buf if cur_staged[1] > 0 else -1
        if pending is not None:
            yield self._result(pending) if pending >= 0 else (0, 0, 0.0, 0, 0, 0)

    def train_chunk(self, ids_host, offsets_host, token_base: int, epoch: int = 0,
                    words_base: int | None = None):
        """One chunk, synchronously (see train_chunks for the pipelined form)."""
        wb = token_base if words_base is None else words_base
        return next(iter(self.train_chunks([(ids_host, offsets_host, token_base, epoch, wb)])))
