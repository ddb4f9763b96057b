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
    # new (device transports only): average only the selected rows that some rank wrote
    # since that row was last averaged.  A row no rank touched holds the same value on
    # every replica, so its mean is itself: the result equals averaging every selected row
    # (bit for bit when the rank count is a power of two, where x * N / N is exact).
    touched_rows: bool = False

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


def _coalescing(dist, group, device):
    """ncclGroupStart/End around the enclosed collectives (torch's coalescing manager).
    async_ops=False: on exit the group's work is waited, i.e. the current CUDA stream is
    made to wait for NCCL's, so the next training launch cannot overlap the average (with
    async_ops=True torch leaves that wait to the caller)."""
    from torch.distributed.distributed_c10d import _coalescing_manager
    return _coalescing_manager(group=group, device=device, async_ops=False)


class NcclTransport(Transport):
    """torch.distributed collective: NCCL over NVLink/NVSwitch on GPUs, gloo on CPU.

    Implements the reference contract (sgns/distributed.py:114-136) for device tensors
    and numpy matrices alike, plus three device-side extensions distributed_train uses:
      * average_rows: both matrices' row slices in ONE coalesced group (ncclGroupStart/
        End; a (2, V, ld) model storage and a full-row set make it one all_reduce);
      * union_flags: OR of per-rank touched-row maps (all_reduce MAX on uint8);
      * average_packed: rows gathered into one buffer, averaged, scattered back.
    precision="native" averages in the model dtype (NCCL AVG); "float64" sums float32
    rows in float64 and rounds the mean once, as the reference's in-process and TCP
    transports accumulate (2x the bytes on the wire).
    """

    MAX_SLICES = 4
    device_native = True

    def __init__(self, group=None, precision: str = "native"):
        import torch.distributed as dist
        if not dist.is_initialized():
            raise TransportError("torch.distributed is not initialised")
        if precision not in ("native", "float64"):
            raise ValueError(f"unknown precision {precision!r}")
        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.nodes = dist.get_world_size(group)
        self.backend = dist.get_backend(group)
        self.precision = precision

    def barrier(self) -> None:
        try:
            self.dist.barrier(group=self.group)
        except Exception as exc:  # noqa: BLE001 - backend errors vary by backend
            raise TransportError(f"barrier failed: {exc}") from exc

    # -- primitives -----------------------------------------------------------
    def _widen(self, t):
        import torch
        return self.precision == "float64" and t.dtype == torch.float32

    def _reduce_many(self, tensors) -> None:
        """In-place mean of each tensor across ranks, as one coalesced group on NCCL."""
        dist = self.dist
        tensors = [t for t in tensors if t.numel()]
        if not tensors:
            return
        work = [t.double() if self._widen(t) else t for t in tensors]
        nccl = self.backend == "nccl"
        op = dist.ReduceOp.AVG if nccl and not any(self._widen(t) for t in tensors) else dist.ReduceOp.SUM
        if nccl and len(work) > 1:
            with _coalescing(dist, self.group, work[0].device):
                for w in work:
                    dist.all_reduce(w, op=op, group=self.group)
        else:
            for w in work:
                dist.all_reduce(w, op=op, group=self.group)
        for t, w in zip(tensors, work):
            if op == dist.ReduceOp.SUM:
                w.div_(self.nodes)
            if w is not t:
                t.copy_(w)

    def _wrap(self, what: str, fn) -> None:
        try:
            fn()
        except TransportError:
            raise
        except Exception as exc:  # noqa: BLE001
            raise TransportError(f"{what} failed: {exc}") from exc

    # -- reference contract --------------------------------------------------
    def allreduce_average(self, matrix, row_ids, which: str) -> None:
        import torch
        if which not in ("in", "out"):
            raise ValueError(f"unknown matrix selector {which!r}")
        if self.nodes == 1:
            return
        host = isinstance(matrix, np.ndarray)
        t = torch.from_numpy(matrix) if host else matrix
        if host and self.backend == "nccl":  # a numpy matrix (reference-style caller)
            dev = torch.device("cuda", torch.cuda.current_device())
            rows = torch.as_tensor(np.asarray(row_ids, dtype=np.int64))
            buf = t.index_select(0, rows).to(dev)
            self._wrap(f"allreduce of {which!r} rows", lambda: self._reduce_many([buf]))
            t.index_copy_(0, rows, buf.cpu())
            return
        self._wrap(f"allreduce of {which!r} rows", lambda: self._average_rows_one(t, row_ids))

    def _average_rows_one(self, t, row_ids) -> None:
        import torch
        runs = row_runs(np.asarray(row_ids, dtype=np.int64))
        if len(runs) <= self.MAX_SLICES:
            self._reduce_many([t[lo:hi] for lo, hi in runs])
        else:
            idx = torch.as_tensor(np.asarray(row_ids, dtype=np.int64), device=t.device)
            buf = t.index_select(0, idx)
            self._reduce_many([buf])
            t.index_copy_(0, idx, buf)

    # -- device extensions ----------------------------------------------------
    def average_rows(self, model, row_ids) -> None:
        """Average the same rows of M_in and M_out in one coalesced group."""
        if self.nodes == 1:
            return
        runs = row_runs(np.asarray(row_ids, dtype=np.int64))
        V = model.m_in.shape[0]
        st = getattr(model, "storage", None)

        def go():
            if st is not None and runs == [(0, V)]:
                self._reduce_many([st])  # the whole model: one all_reduce
            elif len(runs) <= self.MAX_SLICES:
                self._reduce_many([m[lo:hi] for m in (model.m_in, model.m_out) for lo, hi in runs])
            else:
                self._average_rows_one(model.m_in, row_ids)
                self._average_rows_one(model.m_out, row_ids)
        self._wrap("row average", go)

    def union_flags(self, flags) -> None:
        """flags (uint8, any shape) <- elementwise OR over ranks."""
        if self.nodes == 1:
            return
        self._wrap("flag union", lambda: self.dist.all_reduce(flags, op=self.dist.ReduceOp.MAX,
                                                              group=self.group))

    def average_packed(self, parts) -> None:
        """parts: [(matrix, row_index_tensor)]: gather every part's rows into one buffer,
        average it with one collective, scatter the means back."""
        import torch
        if self.nodes == 1:
            return
        parts = [(m, i) for m, i in parts if i.numel()]
        if not parts:
            return
        bufs = [m.index_select(0, i) for m, i in parts]
        flat = torch.cat([b.reshape(-1) for b in bufs])
        self._wrap("packed row average", lambda: self._reduce_many([flat]))
        o = 0
        for (m, i), b in zip(parts, bufs):
            n = b.numel()
            m.index_copy_(0, i, flat[o:o + n].view_as(b))
            o += n

    def close(self) -> None:
        pass


class HostStagedTransport(Transport):
    """Adapter for transports written against the reference contract, which average rows
    of a host numpy matrix (sgns/distributed.py:114-136; its TCP and in-process transports,
    or any user object).  Per call the selected rows of the device matrix are copied into a
    persistent (V, D) host mirror, the wrapped transport averages them there, and they are
    copied back.  Exceptions other than TransportError are re-raised as TransportError, so
    distributed_train reports them as DistributedRunError with partial stats."""

    device_native = False

    def __init__(self, inner, dim: int):
        self.inner = inner
        self.dim = dim
        self.rank = inner.rank
        self.nodes = inner.nodes
        self._mirror: dict = {}

    def barrier(self) -> None:
        try:
            self.inner.barrier()
        except TransportError:
            raise
        except Exception as exc:  # noqa: BLE001
            raise TransportError(f"barrier failed: {exc}") from exc

    def allreduce_average(self, matrix, row_ids, which: str) -> None:
        import torch
        V = matrix.shape[0]
        np_dt = np.float64 if matrix.dtype == torch.float64 else np.float32
        mir = self._mirror.get(which)
        if mir is None or mir.shape != (V, self.dim) or mir.dtype != np_dt:
            mir = self._mirror[which] = np.zeros((V, self.dim), dtype=np_dt)
        rows = np.asarray(row_ids, dtype=np.int64)
        runs = row_runs(rows)
        view = matrix[:, :self.dim]
        for lo, hi in runs:
            mir[lo:hi] = view[lo:hi].cpu().numpy()
        try:
            self.inner.allreduce_average(mir, rows, which)
        except TransportError:
            raise
        except Exception as exc:  # noqa: BLE001
            raise TransportError(f"transport failed averaging {which!r} rows: {exc}") from exc
        for lo, hi in runs:
            view[lo:hi].copy_(torch.from_numpy(mir[lo:hi]))

    def close(self) -> None:
        self.inner.close()


class DistributedRunError(RuntimeError):
    """Training aborted mid-run; carries whatever stats were gathered."""

    def __init__(self, message: str, partial_stats: TrainingStats) -> None:
        super().__init__(message)
        self.partial_stats = partial_stats


def _device_run(vocab, encoded, config, alpha0_eff, total_x_epochs, sent_range, rank, device,
                track_dirty=False):
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
                     sent_range=sent_range, stream_base=rank * n_workers, track_dirty=track_dirty)


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
    device_tr = getattr(transport, "device_native", False)
    tr = transport if device_tr else HostStagedTransport(transport, config.dim)
    if policy.touched_rows and not (device_tr and hasattr(transport, "union_flags")):
        raise ValueError("touched_rows sync needs a device transport (NcclTransport)")
    shards = partition_corpus(encoded, nodes)
    shard_tokens = [int(encoded.offsets[hi] - encoded.offsets[lo]) for lo, hi in shards]
    rounds = max(math.ceil(t * config.epochs / policy.period_words) for t in shard_tokens)
    alpha0_eff = scaled_alpha0(config.alpha0, nodes)
    total_x_epochs = float(encoded.n_tokens) * config.epochs / nodes
    if run_factory is None:
        factory = lambda *a: _device_run(*a, device, track_dirty=policy.touched_rows)  # noqa: E731
    else:
        factory = run_factory
    run = factory(vocab, encoded, config, alpha0_eff, total_x_epochs, shards[transport.rank],
                  transport.rank)
    if policy.touched_rows and getattr(run, "dirty", None) is None:
        raise ValueError("touched_rows sync needs an engine that records touched rows")
    worker_budget = math.ceil(policy.period_words / run.n_workers)
    all_rows = np.arange(vocab.size, dtype=np.int64)
    model = run.model
    started = time.perf_counter()

    def sync(row_ids) -> None:
        if policy.touched_rows:
            sync_touched(row_ids)
        elif hasattr(tr, "average_rows"):
            tr.average_rows(model, row_ids)
        else:
            tr.allreduce_average(model.m_in, row_ids, "in")
            tr.allreduce_average(model.m_out, row_ids, "out")

    def sync_touched(row_ids) -> None:
        import torch
        dirty = run.dirty  # (2, V) uint8: rows written since they were last averaged
        tr.union_flags(dirty)
        parts = []
        for w, m in enumerate((model.m_in, model.m_out)):
            idx = [torch.nonzero(dirty[w, lo:hi]).flatten() + lo for lo, hi in row_runs(row_ids)]
            parts.append((m, torch.cat(idx) if idx else dirty.new_zeros(0, dtype=torch.int64)))
        tr.average_packed(parts)
        for lo, hi in row_runs(row_ids):
            dirty[:, lo:hi] = 0

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
