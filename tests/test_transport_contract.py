"""The reference's pluggable Transport contract (sgns/distributed.py:114-136) behind
distributed_train, on CPU (the oracle is each rank's engine, tests/test_distributed_gloo.py):

* a transport written against the reference -- plain numpy matrices, no torch -- plugs in
  unchanged: distributed_train host-stages the selected rows through it
  (HostStagedTransport), and a two-thread numpy transport reproduces the reference's own
  in-process N = 2 result (tests/golden/dist.npz) bit for bit;
* the failure path: a transport that raises mid-run surfaces as DistributedRunError
  carrying partial stats with words_processed > 0 (the reference's FailingTransport,
  tests/test_distributed.py:206-223), whether it raises TransportError or anything else.
"""

import threading

import numpy as np
import pytest

from helpers import load_golden
from test_distributed_gloo import OracleEngine


class ThreadGroup:
    def __init__(self, nodes):
        self.nodes = nodes
        self.bar = threading.Barrier(nodes)
        self.rows = [None] * nodes


def _numpy_transport_cls():
    from paper_1604_04661_b200.distributed import Transport

    class NumpyThreadTransport(Transport):
        """Reference-contract transport over numpy only: every rank deposits its rows,
        then each computes the rank-order float64 mean itself."""

        def __init__(self, group, rank):
            self.g, self.rank, self.nodes = group, rank, group.nodes
            self.calls = 0

        def barrier(self):
            self.g.bar.wait()

        def allreduce_average(self, matrix, row_ids, which):
            assert isinstance(matrix, np.ndarray) and matrix.flags.c_contiguous
            self.calls += 1
            rows = np.asarray(row_ids, dtype=np.int64)
            self.g.rows[self.rank] = matrix[rows].astype(np.float64)
            self.g.bar.wait()
            acc = self.g.rows[0].copy()
            for r in range(1, self.nodes):
                acc += self.g.rows[r]
            self.g.bar.wait()
            matrix[rows] = (acc / self.nodes).astype(matrix.dtype)

    return NumpyThreadTransport


def _dist_inputs():
    import paper_1604_04661_b200 as P
    from paper_1604_04661_b200.corpus import EncodedCorpus, Vocabulary
    g = load_golden("train")
    enc = EncodedCorpus(g["ids"], g["offsets"], g["sentence_bytes"])
    vocab = Vocabulary.from_counts(g["counts"])
    cfg = P.TrainingConfig(dim=8, window=3, negatives=3, subsample=1e-3, min_count=1, epochs=2,
                           threads=1, seed=4, float64=True, rng="splitmix")
    pol = P.SyncPolicy(period_words=4000, hot_rows=20, rotation_chunk=30)
    return vocab, enc, cfg, pol


def test_numpy_transport_reproduces_reference_two_ranks():
    import paper_1604_04661_b200 as P
    vocab, enc, cfg, pol = _dist_inputs()
    cls = _numpy_transport_cls()
    group = ThreadGroup(2)
    trs = [cls(group, r) for r in range(2)]
    out = [None, None]
    errs = []

    def rank_main(r):
        try:
            out[r] = P.distributed_train(None, cfg, pol, trs[r], prebuilt=(vocab, enc),
                                         run_factory=OracleEngine)
        except BaseException as exc:  # noqa: BLE001
            errs.append(exc)
            group.bar.abort()

    ts = [threading.Thread(target=rank_main, args=(r,)) for r in range(2)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert not errs, errs
    d = load_golden("dist")
    (m0, s0), (m1, s1) = out
    assert trs[0].calls > 2
    assert np.array_equal(m0[0], m1[0]) and np.array_equal(m0[1], m1[1])
    assert np.array_equal(m0[0], d["dp2_min"])
    assert np.array_equal(m0[1], d["dp2_mout"])
    st = d["dp2_stats"]
    assert [s0.words_processed, s0.words_read] == st[:2].tolist()
    assert [s1.words_processed, s1.words_read] == st[2:].tolist()


@pytest.mark.parametrize("exc_kind", ["transport", "other"])
def test_failing_transport_carries_partial_stats(exc_kind):
    import paper_1604_04661_b200 as P
    from paper_1604_04661_b200.distributed import DistributedRunError, Transport, TransportError

    class FailingTransport(Transport):
        rank = 0
        nodes = 1

        def barrier(self):
            pass

        def allreduce_average(self, matrix, row_ids, which):
            if exc_kind == "transport":
                raise TransportError("synthetic link loss")
            raise OSError("socket reset")

    vocab, enc, cfg, _ = _dist_inputs()
    policy = P.SyncPolicy(period_words=20, hot_rows=2, rotation_chunk=1)
    with pytest.raises(DistributedRunError) as info:
        P.distributed_train(None, cfg, policy, FailingTransport(), prebuilt=(vocab, enc),
                            run_factory=OracleEngine)
    assert info.value.partial_stats.words_processed > 0
    assert info.value.partial_stats.words_read > 0


def test_touched_rows_need_a_device_transport():
    import paper_1604_04661_b200 as P
    vocab, enc, cfg, _ = _dist_inputs()
    cls = _numpy_transport_cls()
    tr = cls(ThreadGroup(1), 0)
    with pytest.raises(ValueError):
        P.distributed_train(None, cfg, P.SyncPolicy(touched_rows=True), tr, prebuilt=(vocab, enc),
                            run_factory=OracleEngine)
