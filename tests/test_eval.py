"""Evaluation against the reference's eval_similarity / eval_analogy
on the same vectors and files (header line, OOV and lowercase fallbacks, sections,
max_vocab, a zero row).  Similarity also runs on the host; analogy is a device GEMM."""

import numpy as np
import pytest

from helpers import load_golden

from paper_1604_04661_b200.corpus import Vocabulary
from paper_1604_04661_b200.evaluate import (EvalDataError, eval_analogy, eval_similarity, rank_average,
                                            spearman)
from paper_1604_04661_b200.model import EmbeddingModel


def _setup(tmp_path):
    g = load_golden("eval_full")
    toks = str(g["tokens"]).split("\x00")
    voc = Vocabulary(toks, np.arange(len(toks), 0, -1, dtype=np.int64), {t: i for i, t in enumerate(toks)}, 1)
    sim, ana = tmp_path / "sim.txt", tmp_path / "ana.txt"
    sim.write_text(str(g["sim"]))
    ana.write_text(str(g["ana"]))
    return g, EmbeddingModel(g["vecs"], np.zeros_like(g["vecs"])), voc, str(sim), str(ana)


def test_similarity_matches_reference(tmp_path):
    g, model, voc, sim, _ = _setup(tmp_path)
    rho, used, skipped = eval_similarity(model, voc, sim)
    assert [used, skipped] == g["sim_out"][1:].astype(int).tolist()
    assert rho == pytest.approx(float(g["sim_out"][0]), abs=1e-9)


def test_rank_statistics():
    rng = np.random.default_rng(0)
    for _ in range(20):
        v = rng.integers(0, 5, size=int(rng.integers(2, 30))).astype(float)
        brute = np.array([np.mean([1 + j for j in range(len(v)) if sorted(v)[j] == x]) for x in v])
        assert np.array_equal(rank_average(v), brute)
    assert spearman([1, 2, 3], [10, 20, 30]) == pytest.approx(1.0)
    with pytest.raises(ValueError):
        spearman([1.0], [2.0])


def test_missing_pairs_raise(tmp_path):
    g, model, voc, _, _ = _setup(tmp_path)
    p = tmp_path / "oov.txt"
    p.write_text("zzz yyy 1.0\n")
    with pytest.raises(EvalDataError):
        eval_similarity(model, voc, str(p))


@pytest.mark.gpu
def test_analogy_matches_reference(tmp_path):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("needs CUDA")
    g, model, voc, _, ana = _setup(tmp_path)
    acc, by_sec, skipped = eval_analogy(model, voc, ana)
    acc2, by_sec2, skipped2 = eval_analogy(model, voc, ana, max_vocab=250, block=64)
    assert acc == pytest.approx(float(g["ana_out"][0]), abs=1e-12) and skipped == int(g["ana_out"][1])
    assert acc2 == pytest.approx(float(g["ana_out"][2]), abs=1e-12) and skipped2 == int(g["ana_out"][3])
    for k in range(4):
        assert list(by_sec[f"section{k}"]) + list(by_sec2[f"section{k}"]) == g["ana_sec"][k].tolist()
    from paper_1604_04661_b200.model import DeviceModel
    acc3, _, _ = eval_analogy(DeviceModel.from_host(model), voc, ana)
    assert acc3 == acc


@pytest.mark.gpu
@pytest.mark.parametrize("dim", [1, 7, 8, 100, 128, 129, 300, 517])
def test_unit_rows_bit_identical_to_numpy(dim):
    """sgns_unit_rows == vectors / np.linalg.norm(vectors, axis=1) (zero norm -> 1) bit for
    bit: numpy's pairwise float32 summation order, across its 8 / 128 / halving regimes."""
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("needs CUDA")
    from paper_1604_04661_b200.evaluate import unit_rows
    rng = np.random.default_rng(dim)
    v = (rng.normal(size=(333, dim)) * 10.0 ** rng.integers(-3, 3, size=(333, 1))).astype(np.float32)
    v[5] = 0.0
    norms = np.linalg.norm(v, axis=1, keepdims=True)
    norms[norms == 0.0] = 1.0
    want = v / norms
    got = unit_rows(torch.from_numpy(v).cuda(), dim, len(v)).cpu().numpy()
    assert np.array_equal(got.view(np.uint32), want.view(np.uint32))


@pytest.mark.gpu
@pytest.mark.parametrize("n,dim,nq", [(5, 3, 4), (1000, 300, 257), (40_000, 100, 1500)])
def test_analogy_top1_vs_brute_force(n, dim, nq):
    """The fused score/argmax kernel against a float64 brute force: the same row except where
    the float64 top two lie within float32 rounding of each other (a legal tie flip)."""
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("needs CUDA")
    from paper_1604_04661_b200.evaluate import analogy_top1
    rng = np.random.default_rng(n + dim)
    u = rng.normal(size=(n, dim)).astype(np.float32)
    u /= np.linalg.norm(u, axis=1, keepdims=True)
    q = np.stack([rng.choice(n, size=3, replace=False) for _ in range(nq)]).astype(np.int32)
    got = analogy_top1(torch.from_numpy(u).cuda(), q)
    t = (u[q[:, 1]] - u[q[:, 0]] + u[q[:, 2]]).astype(np.float64)
    s = t @ u.astype(np.float64).T
    s[np.arange(nq)[:, None], q] = -np.inf
    want = s.argmax(axis=1)
    top = np.sort(s, axis=1)[:, -2:]
    close = (top[:, 1] - top[:, 0]) < 1e-5 * np.abs(top[:, 1]).clip(1.0)
    bad = (got != want) & ~close
    assert not bad.any(), np.flatnonzero(bad)[:5]
    assert (got == want).mean() > 0.99
    assert not (got[:, None] == q).any()  # never a question word
