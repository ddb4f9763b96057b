"""Data-parallel training: one process per GPU, NCCL row averaging over NVLink.

Reference map:
  TransportError / HandshakeError  sgns/distributed.py:46-51
  SyncPolicy                       sgns/distributed.py:54-83
  select_sync_rows                 sgns/distributed.py:86-101
  scaled_alpha0                    sgns/distributed.py:104-106
  partition_corpus                 sgns/distributed.py:109-111 (-> partition_sentences)
  Transport contract               sgns/distributed.py:114-136
  DistributedRunError              sgns/distributed.py:406-411
  distributed_train                sgns/distributed.py:421-512

Each rank trains its byte-balanced shard on its own GPU with the device driver
and, every `period_words` words read, averages the hot rows [0, F) plus one
round-robin chunk of both matrices.  Vocabulary ids are frequency sorted, so
the selected rows are at most two contiguous slices per matrix and
`NcclTransport` averages them in place with `all_reduce(AVG)` on row slices --
no gather/scatter.  The all-gather phase of the collective leaves replicas
bit-identical, as the reference requires (tests/test_distributed.py:119-124).
"""

from __future__ import annotations

import math
import time
from dataclasses import dataclass, replace

import numpy as np

from .corpus import EncodedCorpus, Vocabulary, build_vocab, encode_corpus, partition_sentences, read_tokens
from .trainer import (DeviceCorpus, DeviceRun, DeviceSampler, TrainingConfig, TrainingStats,
                      default_workers, update_alpha)


class TransportError(RuntimeError):
    """Collective communication failed."""


class HandshakeError(TransportError):
    """Peers disagree on geometry or configuration."""


@dataclass
class SyncPolicy:
    period_words: int = 1_000_000
    hot_rows: int | None = None
    rotation_chunk: int | None = None

    def resolve(self, vocab_size: int) -> "SyncPolicy":
        hot = self.hot_rows if self.hot_rows is not None else min(vocab_size, 10_000)
        cold = vocab_size - hot
        if self.rotation_chunk is not None:
            rot = self.rotation_chunk
        else:
            rot = math.ceil(cold / 20) if cold else 0
        policy = replace(self, hot_rows=hot, rotation_chunk=rot)
        policy.validate(vocab_size)
        return policy

    def validate(self, vocab_size: int) -> None:
        if self.period_words < 1:
            raise ValueError("period_words must be >= 1")
        if not 0 <= self.hot_rows <= vocab_size:
            raise ValueError("hot_rows must be in [0, vocab_size]")
        if not 0 <= self.rotation_chunk <= vocab_size - self.hot_rows:
            raise ValueError("rotation_chunk must be in [0, vocab_size - hot_rows]")


def sync_row_ranges(vocab_size: int, policy: SyncPolicy, period_index: int) -> list[tuple[int, int]]:
    """The rows of select_sync_rows as at most two [lo, hi) slices."""
    policy = policy.resolve(vocab_size)
    hot, rot = policy.hot_rows, policy.rotation_chunk
    cold = vocab_size - hot
    out = [(0, hot)] if hot else []
    if rot == 0 or cold == 0:
        return out
    n_chunks = math.ceil(cold / rot)
    start = hot + (period_index % n_chunks) * rot
    stop = min(start + rot, vocab_size)
    if out and out[-1][1] == start:
        out[-1] = (out[-1][0], stop)
    else:
        out.append((start, stop))
    return out


def select_sync_rows(vocab_size: int, policy: SyncPolicy, period_index: int) -> np.ndarray:
    """Row ids to average this period: hot rows plus one round-robin chunk."""
    ranges = sync_row_ranges(vocab_size, policy, period_index)
    if not ranges:
        return np.empty(0, dtype=np.int64)
    return np.concatenate([np.arange(a, b, dtype=np.int64) for a, b in ranges])


def scaled_alpha0(alpha0: float, nodes: int) -> float:
    return alpha0 * math.sqrt(nodes)


def partition_corpus(encoded: EncodedCorpus, nodes: int) -> list[tuple[int, int]]:
    return partition_sentences(encoded, nodes)


def row_runs(row_ids: np.ndarray) -> list[tuple[int, int]]:
    """Maximal contiguous [lo, hi) runs of a sorted row-id vector."""
    r = np.asarray(row_ids, dtype=np.int64)
    if r.size == 0:
        return []
    brk = np.flatnonzero(np.diff(r) != 1) + 1
    starts = np.concatenate([[0], brk])
    stops = np.concatenate([brk, [r.size]])
    return [(int(r[a]), int(r[b - 1]) + 1) for a, b in zip(starts, stops)]


class Transport:
    """Collective operations over N replicas (sgns/distributed.py:114-136)."""

    rank: int
    nodes: int

    def barrier(self) -> None:
        raise NotImplementedError

    def allreduce_average(self, matrix, row_ids, which: str) -> None:
        raise NotImplementedError

    def close(self) -> None:
        pass


class NcclTransport(Transport):
    """torch.distributed collective: NCCL over NVLink/NVSwitch on GPUs, gloo on CPU.

    Rows are averaged in place on contiguous slices of the (V, ld) matrix
    (all_reduce AVG on NCCL; SUM then divide on gloo, which lacks AVG).  Row
    sets that are not a few contiguous runs go through one packed buffer.
    """

    MAX_SLICES = 4

    def __init__(self, group=None):
        import torch.distributed as dist
        if not dist.is_initialized():
            raise TransportError("torch.distributed is not initialised")
        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.nodes = dist.get_world_size(group)
        self.backend = dist.get_backend(group)

    def barrier(self) -> None:
        try:
            self.dist.barrier(group=self.group)
        except Exception as exc:  # noqa: BLE001 - backend errors vary by backend
            raise TransportError(f"barrier failed: {exc}") from exc

    def _reduce(self, t) -> None:
        dist = self.dist
        if self.backend == "nccl":
            dist.all_reduce(t, op=dist.ReduceOp.AVG, group=self.group)
        else:
            dist.all_reduce(t, op=dist.ReduceOp.SUM, group=self.group)
            t.div_(self.nodes)

    def allreduce_average(self, matrix, row_ids, which: str) -> None:
        import torch
        if which not in ("in", "out"):
            raise ValueError(f"unknown matrix selector {which!r}")
        if self.nodes == 1:
            return
        runs = row_runs(np.asarray(row_ids, dtype=np.int64))
        try:
            if len(runs) <= self.MAX_SLICES:
                for lo, hi in runs:
                    self._reduce(matrix[lo:hi])
            else:
                idx = torch.as_tensor(np.asarray(row_ids, dtype=np.int64), device=matrix.device)
                buf = matrix.index_select(0, idx)
                self._reduce(buf)
                matrix.index_copy_(0, idx, buf)
        except TransportError:
            raise
        except Exception as exc:  # noqa: BLE001
            raise TransportError(f"allreduce of {which!r} rows failed: {exc}") from exc

    def close(self) -> None:
        pass


class DistributedRunError(RuntimeError):
    """Training aborted mid-run; carries whatever stats were gathered."""

    def __init__(self, message: str, partial_stats: TrainingStats) -> None:
        super().__init__(message)
        self.partial_stats = partial_stats


def _device_run(vocab, encoded, config, alpha0_eff, total_x_epochs, sent_range, rank, device):
    """Default engine: this rank's shard on its GPU (DeviceRun over W workers)."""
    from .model import init_device_model
    import torch
    if device is None:
        device = torch.device("cuda", torch.cuda.current_device())
    dm = init_device_model(vocab.size, config.dim, config.seed, config.dtype, device)
    corpus = DeviceCorpus(encoded, dm.m_in.device)
    sampler = DeviceSampler(vocab.counts, config.rng, config.table_length, None, dm.m_in.device)
    keep = vocab.keep_probs(config.subsample) if config.subsample > 0 else None
    n_workers = default_workers(config, corpus, sent_range[1] - sent_range[0],
                                int(encoded.offsets[sent_range[1]] - encoded.offsets[sent_range[0]]))
    return DeviceRun(dm, corpus, sampler, keep, config, alpha0_eff, total_x_epochs, n_workers,
                     sent_range=sent_range, stream_base=rank * n_workers)


def distributed_train(corpus_path: str | None, config: TrainingConfig, policy: SyncPolicy,
                      transport: Transport, prebuilt: tuple[Vocabulary, EncodedCorpus] | None = None,
                      *, device=None, run_factory=None, return_device: bool = False):
    """Train this rank's replica; returns (model, stats).  Replicas end identical."""
    config.validate()
    if prebuilt is not None:
        vocab, encoded = prebuilt
    else:
        if corpus_path is None:
            raise ValueError("need a corpus path or a prebuilt (vocab, corpus) pair")
        from .corpus import build_vocab_file, encode_corpus_file
        vocab = build_vocab_file(corpus_path, config.min_count)
        encoded = encode_corpus_file(corpus_path, vocab)
    nodes = transport.nodes
    policy = policy.resolve(vocab.size)
    shards = partition_corpus(encoded, nodes)
    shard_tokens = [int(encoded.offsets[hi] - encoded.offsets[lo]) for lo, hi in shards]
    rounds = max(math.ceil(t * config.epochs / policy.period_words) for t in shard_tokens)
    alpha0_eff = scaled_alpha0(config.alpha0, nodes)
    total_x_epochs = float(encoded.n_tokens) * config.epochs / nodes
    factory = run_factory or (lambda *a: _device_run(*a, device))
    run = factory(vocab, encoded, config, alpha0_eff, total_x_epochs, shards[transport.rank],
                  transport.rank)
    worker_budget = math.ceil(policy.period_words / run.n_workers)
    all_rows = np.arange(vocab.size, dtype=np.int64)
    m_in, m_out = run.model.m_in, run.model.m_out
    started = time.perf_counter()

    def sync(row_ids) -> None:
        transport.allreduce_average(m_in, row_ids, "in")
        transport.allreduce_average(m_out, row_ids, "out")

    def partial_stats() -> TrainingStats:
        stats = TrainingStats()
        stats.words_processed = run.words_trained
        stats.words_read = run.words_read
        stats.wall_seconds = time.perf_counter() - started
        stats.throughput_words_per_sec = stats.words_processed / max(stats.wall_seconds, 1e-9)
        stats.final_alpha = update_alpha(run.shared_words_read(), total_x_epochs, alpha0_eff,
                                         config.alpha_floor_fraction)
        stats.loss_by_epoch = run.loss_by_epoch()
        return stats

    try:
        for period in range(rounds):
            run.launch(worker_budget)
            sync(select_sync_rows(vocab.size, policy, period))
        run.run_to_completion()  # drain any words the round estimate missed
        sync(all_rows)
    except TransportError as exc:
        raise DistributedRunError(str(exc), partial_stats()) from exc
    stats = partial_stats()
    if return_device:
        return run.model, stats
    return run.model.to_host(), stats
