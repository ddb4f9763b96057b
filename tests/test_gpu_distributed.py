"""Data parallel on the device path (one GPU in this pool): an NCCL world of one rank
must be byte-identical to single-node training (the reference's C7a,
tests/test_acceptance.py:315-328), through the same NcclTransport and sync schedule."""

import os
import socket

import numpy as np
import pytest

from helpers import load_golden

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("rng", ["splitmix", "philox"])
def test_nccl_world_of_one_equals_single_node(rng):
    if not torch.cuda.is_available():
        pytest.skip("needs CUDA")
    import torch.distributed as dist
    import paper_1604_04661_b200 as P
    from paper_1604_04661_b200.corpus import EncodedCorpus, Vocabulary
    g = load_golden("train")
    enc = EncodedCorpus(g["ids"], g["offsets"], g["sentence_bytes"])
    vocab = Vocabulary.from_counts(g["counts"])
    cfg = P.TrainingConfig(dim=16, window=3, negatives=3, subsample=1e-3, min_count=1, epochs=2,
                           seed=4, rng=rng, workers=1)
    base, _ = P.train_encoded(vocab, enc, cfg)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(_free_port())
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        tr = P.NcclTransport()
        model, stats = P.distributed_train(None, cfg, P.SyncPolicy(period_words=5000, hot_rows=30,
                                                                   rotation_chunk=40),
                                           tr, prebuilt=(vocab, enc))
    finally:
        dist.destroy_process_group()
    assert np.array_equal(model.input_vectors, base.input_vectors)
    assert np.array_equal(model.output_vectors, base.output_vectors)
    assert stats.words_read == 2 * enc.n_tokens


@pytest.mark.parametrize("schedule,k", [("dynamic", 5), ("static", 5), ("static", 12)])
def test_kernels_mark_touched_rows(schedule, k):
    """The drivers' touched-row map (sgns_drive_params.d_dirty) is exactly the set of input
    rows and output rows (targets + negatives) of the windows they applied."""
    if not torch.cuda.is_available():
        pytest.skip("needs CUDA")
    import paper_1604_04661_b200 as P
    from paper_1604_04661_b200.corpus import EncodedCorpus
    from paper_1604_04661_b200.model import DeviceModel
    from paper_1604_04661_b200.synthetic import make_planted_corpus
    from paper_1604_04661_b200.trainer import DeviceCorpus, DeviceRun, DeviceSampler
    syn = make_planted_corpus(6_000, 3_000, n_clusters=4, cluster_size=5, sentence_len=31, seed=2)
    ids, off, counts = syn.encoded.ids, syn.encoded.offsets, syn.vocab.counts
    V = len(counts)
    cfg = P.TrainingConfig(dim=32, window=4, negatives=k, subsample=0.0, min_count=1, seed=3,
                           epochs=1, rng="philox", workers=1, schedule=schedule)
    dm = DeviceModel.empty(V, 32)
    cap = len(ids) + 16
    run = DeviceRun(dm, DeviceCorpus(EncodedCorpus(ids, off, np.zeros(len(off) - 1, np.int64))),
                    DeviceSampler(counts, "philox"), None, cfg, 0.025, float(off[-1]), 1,
                    trace_cap=cap, track_dirty=True)
    assert run.dynamic == (schedule == "dynamic")
    run.run_to_completion()
    recs, _ = run.trace_records() if run.dynamic else run.worker_trace(0)
    assert len(recs) > 1000
    exp = np.zeros((2, V), np.uint8)
    cap_r = cfg.batch_cap
    for r in recs:
        m = int(r[1])
        exp[0, r[4:4 + m]] = 1
        exp[1, r[4 + cap_r:4 + cap_r + k + 1]] = 1
    got = run.dirty.cpu().numpy()
    assert np.array_equal(got, exp)
    assert exp[0].sum() > 0 and exp[1].sum() > 0
