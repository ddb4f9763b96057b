"""The north-star configuration at full size (BASELINE.json configs[3]: 800M tokens,
1M ids, d=300, w=5, K=5, t=1e-4), checked through properties that do not need a CPU
run of the whole corpus:

* exact parity at full vocabulary: on the first ~1M tokens, the production driver's
  windows (target, inputs, shared negatives, alpha) as a multiset equal the oracle's,
  with keep probabilities from the full 800M-token counts and the 1M-entry alias table;
* schedule independence: every subsample / window / negative draw is keyed by token
  position, so the counters of a whole epoch (words read, words trained, chunks,
  inputs) are identical for 2,368 and 600 workers;
* accounting: words read == tokens; words trained within 6 sigma of sum(count * keep);
* training health: mean loss below the untrained ln 2 and finite model rows.
"""

import math

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from test_gpu_parity import _oracle_philox, _run_driver  # noqa: E402

TOKENS, VOCAB, DIM = 800_000_000, 1_000_000, 300


@pytest.fixture(scope="module")
def big():
    if not torch.cuda.is_available():
        pytest.skip("needs CUDA")
    from paper_1604_04661_b200.synthetic import make_planted_corpus_device
    corpus = make_planted_corpus_device(TOKENS, VOCAB, zipf_s=1.05, min_count=5, seed=1, device="cuda")
    yield corpus
    del corpus
    torch.cuda.empty_cache()


def _cfg(**kw):
    import paper_1604_04661_b200 as P
    base = dict(dim=DIM, window=5, negatives=5, subsample=1e-4, min_count=5, alpha0=0.025, epochs=1,
                seed=1, rng="philox", schedule="dynamic")
    base.update(kw)
    return P.TrainingConfig(**base)


def _counters(run):
    st = run.state()
    return (int(st["words_read"].sum()), int(st["words_trained"].sum()), int(st["kernel_counter"].sum()),
            int(st["inputs"].sum()))


def _full_run(corpus, workers, update):
    from paper_1604_04661_b200.corpus import EncodedCorpus, keep_probabilities
    from paper_1604_04661_b200.model import init_device_model
    from paper_1604_04661_b200.trainer import DeviceCorpus, DeviceRun, DeviceSampler
    counts = corpus.counts
    enc = EncodedCorpus(np.empty(0, np.int32), corpus.host_offsets(), corpus.sentence_bytes)
    cfg = _cfg(workers=workers, loss_sample_every=1)
    dcorp = DeviceCorpus(enc, "cuda", ids=corpus.ids, offsets=corpus.offsets)
    model = init_device_model(len(counts), DIM, 1, np.float32, "cuda")
    sampler = DeviceSampler(counts, "philox", device="cuda")
    keep = keep_probabilities(counts, int(counts.sum()), 1e-4)
    run = DeviceRun(model, dcorp, sampler, keep, cfg, 0.025, float(corpus.n_tokens), workers, update=update)
    assert run.dynamic
    run.run_to_completion()
    return run, model


def test_full_vocab_window_stream_matches_oracle(big):
    """First ~1M tokens of the 800M-token corpus, full 1M-id tables: device windows ==
    oracle windows as a multiset, bit for bit (ids, sentence, epoch, alpha)."""
    counts = big.counts
    off_all = big.host_offsets()
    S = int(np.searchsorted(off_all, 1_000_000))
    ids = big.ids[:off_all[S]].cpu().numpy()
    off = off_all[:S + 1].astype(np.int64)
    cap = len(ids) * 2 + 10
    run, sampler = _run_driver(ids, off, counts, window=5, k=5, cap=16, dynamic=True, subsample=1e-4,
                               seed=1, stream_base=0, table_len=None, rng="philox", workers=300,
                               epochs=1, trace_cap=cap, schedule="dynamic", dim=DIM)
    got, got_alpha = run.trace_records()
    orc = _oracle_philox(ids, off, counts, sampler.host_alias, W=1, epochs=1, update=False,
                         trace_cap=cap, cap=16, sub=1e-4, seed=1)
    exp, exp_alpha = orc.worker_trace(0)
    assert len(exp) > 250_000 and got.shape == exp.shape
    key = lambda a, al: np.lexsort(np.column_stack([a, al.view(np.int64)]).T[::-1])
    gi, ei = key(got, got_alpha), key(exp, exp_alpha)
    assert np.array_equal(got[gi], exp[ei])
    assert np.array_equal(got_alpha[gi], exp_alpha[ei])
    assert run.words_trained == orc.workers[0].words_trained
    # negatives reach deep into the 1M-id table (alias draws are not truncated)
    assert exp[:, 4 + 16 + 1:].max() > 500_000


def test_full_epoch_counters_schedule_independent_and_healthy(big):
    counts = big.counts.astype(np.float64)
    run, model = _full_run(big, 2368, update=True)
    a = _counters(run)
    loss = run.loss_by_epoch()
    assert a[0] == big.n_tokens  # every sentence claimed exactly once
    from paper_1604_04661_b200.corpus import keep_probabilities
    p = keep_probabilities(big.counts, int(big.counts.sum()), 1e-4)
    mean, var = float((counts * p).sum()), float((counts * p * (1 - p)).sum())
    assert abs(a[1] - mean) < 6 * math.sqrt(var) + 1
    assert 0.0 < loss[0] < math.log(2.0)
    for m in (model.m_in, model.m_out):
        assert bool(torch.isfinite(m[:, :DIM]).all())
    assert float(model.m_out[:, :DIM].abs().max()) > 0.0
    del run, model
    torch.cuda.empty_cache()
    run2, model2 = _full_run(big, 600, update=False)
    assert _counters(run2) == a
