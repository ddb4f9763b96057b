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
