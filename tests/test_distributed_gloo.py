"""Data-parallel host logic on CPU: world_size-2 torch.distributed (gloo) processes.

* NcclTransport row averaging (contiguous slices and packed row sets) under gloo.
* distributed_train end to end with the oracle as each rank's engine (run_factory):
  float64, 2 ranks, the reference's own in-process N=2 result (tests/golden/dist.npz,
  rank-order float64 mean) must be reproduced bit for bit -- shard partition, round
  count, per-rank alpha0*sqrt(N), budgets, sync row selection and the final average.
"""

import os
import socket
import tempfile

import numpy as np
import pytest

import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from helpers import ROOT, load_golden


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _init(rank, world, port):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)


def _transport_worker(rank, world, port, out):
    import sys
    sys.path.insert(0, ROOT)
    from paper_1604_04661_b200.distributed import NcclTransport
    _init(rank, world, port)
    tr = NcclTransport()
    rng = np.random.default_rng(100 + rank)
    m64 = torch.from_numpy(rng.normal(size=(50, 6)))
    m32 = torch.from_numpy(rng.normal(size=(50, 8)).astype(np.float32))
    tr.allreduce_average(m64, np.arange(10, 25), "in")            # one slice
    tr.allreduce_average(m32, np.array([0, 3, 4, 9, 11, 30, 31, 40, 49]), "out")  # packed
    tr.barrier()
    np.savez(f"{out}_{rank}.npz", m64=m64.numpy(), m32=m32.numpy())
    dist.destroy_process_group()


def test_transport_average_gloo(tmp_path):
    port = _free_port()
    out = str(tmp_path / "tr")
    mp.spawn(_transport_worker, args=(2, port, out), nprocs=2, join=True)
    r = [np.load(f"{out}_{k}.npz") for k in range(2)]
    orig = []
    for k in range(2):
        rng = np.random.default_rng(100 + k)
        orig.append((rng.normal(size=(50, 6)), rng.normal(size=(50, 8)).astype(np.float32)))
    rows64 = np.arange(10, 25)
    expect64 = (orig[0][0][rows64] + orig[1][0][rows64]) / 2
    for k in range(2):
        assert np.array_equal(r[k]["m64"][rows64], expect64)          # 2 ranks: f64 mean exact
        other = np.setdiff1d(np.arange(50), rows64)
        assert np.array_equal(r[k]["m64"][other], orig[k][0][other])  # untouched
    rows32 = np.array([0, 3, 4, 9, 11, 30, 31, 40, 49])
    exp32 = (orig[0][1][rows32].astype(np.float64) + orig[1][1][rows32]) / 2
    assert np.array_equal(r[0]["m32"][rows32], r[1]["m32"][rows32])    # replicas identical
    np.testing.assert_allclose(r[0]["m32"][rows32], exp32, rtol=1e-6)


class OracleEngine:
    """Per-rank engine for distributed_train backed by the C oracle (CPU, tests only)."""

    def __init__(self, vocab, encoded, config, alpha0_eff, total_x_epochs, sent_range, rank):
        from oracle import oracle as O
        from paper_1604_04661_b200.corpus import default_table_length, keep_probabilities
        from paper_1604_04661_b200.model import SIGMOID_TABLE_F32, SIGMOID_TABLE_F64
        V, D = vocab.size, config.dim
        dt = np.float64 if config.float64 else np.float32
        self.m_in_np = O.init_model(V, D, config.seed).astype(dt)
        self.m_out_np = np.zeros((V, D), dt)
        L = config.table_length or default_table_length(V)
        slots = np.repeat(np.arange(V, dtype=np.int32),
                          np.diff(O.neg_boundaries(vocab.counts, 0.75, L), prepend=0))
        keep = keep_probabilities(vocab.counts, vocab.total_tokens, config.subsample) if config.subsample > 0 else None
        self.n_workers = config.threads
        self.run = O.OracleRun(encoded.ids, encoded.offsets, self.m_in_np, self.m_out_np,
                               keep_probs=keep, window=config.window, negatives=config.negatives,
                               batch_cap=config.batch_cap, dynamic=config.dynamic_window,
                               seed=config.seed, alpha0=alpha0_eff,
                               floor_frac=config.alpha_floor_fraction, total_x_epochs=total_x_epochs,
                               epochs=config.epochs, loss_every=config.loss_sample_every,
                               n_workers=self.n_workers, sent_range=sent_range,
                               stream_base=rank * self.n_workers, slots=slots,
                               sig_table=SIGMOID_TABLE_F64 if config.float64 else SIGMOID_TABLE_F32)

        class _M:
            pass
        self.model = _M()
        self.model.m_in = torch.from_numpy(self.m_in_np)
        self.model.m_out = torch.from_numpy(self.m_out_np)
        self.model.to_host = lambda: (self.m_in_np.copy(), self.m_out_np.copy())

        # touched-row map for SyncPolicy(touched_rows=True): the oracle marks rows whose
        # value changed in a launch (a touched row left unchanged averages to itself too)
        self.dirty = torch.zeros((2, V), dtype=torch.uint8)

    def _mark(self, fn):
        before = (self.m_in_np.copy(), self.m_out_np.copy())
        fn()
        for w, (old, new) in enumerate(zip(before, (self.m_in_np, self.m_out_np))):
            changed = torch.from_numpy((old != new).any(axis=1).astype(np.uint8))
            self.dirty[w] |= changed

    def launch(self, budget):
        self._mark(lambda: self.run.advance(budget))

    def run_to_completion(self):
        self._mark(self.run.run_to_completion)

    @property
    def words_trained(self):
        return self.run.stats()[0]

    @property
    def words_read(self):
        return self.run.stats()[1]

    def loss_by_epoch(self):
        return self.run.stats()[2]

    def shared_words_read(self):
        return int(self.run.shared[0])


def _dp_worker(rank, world, port, out):
    import sys
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import paper_1604_04661_b200 as P
    from paper_1604_04661_b200.corpus import EncodedCorpus, Vocabulary
    _init(rank, world, port)
    g = load_golden("train")
    enc = EncodedCorpus(g["ids"], g["offsets"], g["sentence_bytes"])
    vocab = Vocabulary.from_counts(g["counts"])
    cfg = P.TrainingConfig(dim=8, window=3, negatives=3, subsample=1e-3, min_count=1, epochs=2,
                           threads=1, seed=4, float64=True, rng="splitmix")
    pol = P.SyncPolicy(period_words=4000, hot_rows=20, rotation_chunk=30)
    (m_in, m_out), stats = P.distributed_train(None, cfg, pol, P.NcclTransport(), prebuilt=(vocab, enc),
                                               run_factory=OracleEngine)
    np.savez(f"{out}_{rank}.npz", m_in=m_in, m_out=m_out,
             stats=np.array([stats.words_processed, stats.words_read]), loss=np.array(stats.loss_by_epoch))
    dist.destroy_process_group()


def test_distributed_train_two_ranks_matches_reference(tmp_path):
    port = _free_port()
    out = str(tmp_path / "dp")
    mp.spawn(_dp_worker, args=(2, port, out), nprocs=2, join=True)
    d = load_golden("dist")
    r = [np.load(f"{out}_{k}.npz") for k in range(2)]
    assert np.array_equal(r[0]["m_in"], r[1]["m_in"]) and np.array_equal(r[0]["m_out"], r[1]["m_out"])
    assert np.array_equal(r[0]["m_in"], d["dp2_min"])
    assert np.array_equal(r[0]["m_out"], d["dp2_mout"])
    st = d["dp2_stats"]
    assert r[0]["stats"].tolist() == st[:2].tolist()
    assert r[1]["stats"].tolist() == st[2:].tolist()
    np.testing.assert_allclose(r[0]["loss"], d["dp2_loss0"], rtol=1e-12)


def _touched_worker(rank, world, port, out, touched, hot, rot, f64):
    import sys
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import paper_1604_04661_b200 as P
    from paper_1604_04661_b200.corpus import EncodedCorpus, Vocabulary
    _init(rank, world, port)
    g = load_golden("train")
    enc = EncodedCorpus(g["ids"], g["offsets"], g["sentence_bytes"])
    vocab = Vocabulary.from_counts(g["counts"])
    cfg = P.TrainingConfig(dim=8, window=3, negatives=3, subsample=1e-3, min_count=1, epochs=2,
                           threads=1, seed=4, float64=f64, rng="splitmix")
    pol = P.SyncPolicy(period_words=1500, hot_rows=hot, rotation_chunk=rot, touched_rows=touched)
    tr = P.NcclTransport()
    calls = []
    orig = tr.average_packed
    tr.average_packed = lambda parts: (calls.append(sum(int(i.numel()) for _, i in parts)), orig(parts))
    (m_in, m_out), stats = P.distributed_train(None, cfg, pol, tr, prebuilt=(vocab, enc),
                                               run_factory=OracleEngine)
    np.savez(f"{out}_{rank}.npz", m_in=m_in, m_out=m_out, packed=np.array(calls, dtype=np.int64))
    dist.destroy_process_group()


@pytest.mark.parametrize("hot,rot,f64", [(None, 0, False), (20, 30, False), (20, 30, True)],
                         ids=["full_f32", "submodel_f32", "submodel_f64"])
def test_touched_row_sync_equals_full_sync(tmp_path, hot, rot, f64):
    """SyncPolicy(touched_rows=True): only rows some rank wrote since their last average go
    on the wire (flag union = all_reduce MAX, one packed collective); at N = 2 the models
    are bit-identical to averaging every selected row."""
    from paper_1604_04661_b200.corpus import Vocabulary
    V = Vocabulary.from_counts(load_golden("train")["counts"]).size
    hot = V if hot is None else hot
    res = {}
    for touched in (False, True):
        port = _free_port()
        out = str(tmp_path / f"t{int(touched)}")
        mp.spawn(_touched_worker, args=(2, port, out, touched, hot, rot, f64), nprocs=2, join=True)
        res[touched] = [np.load(f"{out}_{k}.npz") for k in range(2)]
    for k in range(2):
        assert np.array_equal(res[True][k]["m_in"], res[False][k]["m_in"])
        assert np.array_equal(res[True][k]["m_out"], res[False][k]["m_out"])
    packed = res[True][0]["packed"]
    assert len(packed) > 2
    assert packed.max() <= 2 * V and packed[:-1].mean() < 2 * min(V, hot + rot)  # fewer rows moved
