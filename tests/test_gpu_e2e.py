"""End-to-end quality bar of the north star on the tiny config (BASELINE.json configs[0]):
the production path (philox + alias, ~2,400 concurrent device workers) against the
reference algorithm at threads=1 (the oracle: splitmix stream, slot table, deterministic).

The loss is evaluated on every cell (loss_sample_every=1) on both sides: with thousands
of workers, sampling each worker's every 100th chunk would only sample late training
progress (each worker owns 1/W of the corpus) and bias the mean low.

  per-epoch loss:             |loss_gpu / loss_ref - 1| <= 2%
  planted-cluster Spearman:   |rho_gpu - rho_ref| <= 0.01 (correlation units, mean of 3 seeds)
"""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def tiny():
    if not torch.cuda.is_available():
        pytest.skip("needs CUDA")
    from paper_1604_04661_b200.synthetic import tiny_config_corpus
    return tiny_config_corpus(seed=0)


def _reference_run(syn, seed):
    from oracle import oracle as O
    from paper_1604_04661_b200.corpus import default_table_length, keep_probabilities
    from paper_1604_04661_b200.model import SIGMOID_TABLE_F32
    counts = syn.vocab.counts
    V, D = len(counts), 100
    L = default_table_length(V)
    slots = np.repeat(np.arange(V, dtype=np.int32), np.diff(O.neg_boundaries(counts, 0.75, L), prepend=0))
    m_in = O.init_model(V, D, seed).astype(np.float32)
    m_out = np.zeros((V, D), np.float32)
    run = O.OracleRun(syn.encoded.ids, syn.encoded.offsets, m_in, m_out,
                      keep_probs=keep_probabilities(counts, int(counts.sum()), 1e-4), window=5,
                      negatives=5, batch_cap=16, dynamic=True, seed=seed, alpha0=0.025,
                      floor_frac=1e-4, total_x_epochs=float(syn.encoded.n_tokens), epochs=1,
                      loss_every=1, n_workers=1, slots=slots, sig_table=SIGMOID_TABLE_F32)
    run.run_to_completion()
    return m_in, run.stats()[2][0]


def _gpu_run(syn, seed, **kw):
    import paper_1604_04661_b200 as P
    cfg = P.TrainingConfig(dim=100, window=5, negatives=5, subsample=1e-4, min_count=1,
                           alpha0=0.025, epochs=1, seed=seed, loss_sample_every=1, **kw)
    model, stats = P.train_encoded(syn.vocab, syn.encoded, cfg)
    return model.input_vectors, stats


def _rho(vecs, syn):
    from paper_1604_04661_b200.evaluate import similarity_score
    rho, used, skipped = similarity_score(vecs, syn.vocab.index, syn.gold_pairs(pairs_per_cluster=16))
    assert skipped == 0
    return rho / 100.0


def test_production_path_matches_reference_quality(tiny):
    ref_loss, gpu_loss, ref_rho, gpu_rho = [], [], [], []
    for seed in (1, 2, 3):
        vr, lr = _reference_run(tiny, seed)
        vg, st = _gpu_run(tiny, seed)
        ref_loss.append(lr)
        gpu_loss.append(st.loss_by_epoch[0])
        ref_rho.append(_rho(vr, tiny))
        gpu_rho.append(_rho(vg, tiny))
    rl, gl = float(np.mean(ref_loss)), float(np.mean(gpu_loss))
    rr, gr = float(np.mean(ref_rho)), float(np.mean(gpu_rho))
    print(f"\nE2E tiny: loss ref {rl:.4f} gpu {gl:.4f} ({100 * (gl / rl - 1):+.2f}%); "
          f"rho ref {rr:.4f} gpu {gr:.4f} (diff {gr - rr:+.4f})")
    print("per seed: ref loss", ref_loss, "gpu loss", gpu_loss, "ref rho", ref_rho, "gpu rho", gpu_rho)
    assert abs(gl / rl - 1.0) <= 0.02
    assert abs(gr - rr) <= 0.01


def test_reference_stream_mode_single_worker_matches_reference_loss(tiny):
    """rng='splitmix', workers=1: the exact reference stream; loss within 0.2%."""
    vr, lr = _reference_run(tiny, 1)
    vg, st = _gpu_run(tiny, 1, rng="splitmix", workers=1)
    assert abs(st.loss_by_epoch[0] / lr - 1.0) <= 0.002
    assert abs(_rho(vg, tiny) - _rho(vr, tiny)) <= 0.01
