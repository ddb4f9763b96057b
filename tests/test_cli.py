"""CLI: flags, reports and exit codes as the reference CLI."""

import os
import subprocess
import sys

import numpy as np
import pytest

from helpers import ROOT

from paper_1604_04661_b200.cli import build_parser, main


def _run(*args, env=None):
    return subprocess.run([sys.executable, "-m", "paper_1604_04661_b200", *args], cwd=ROOT,
                          capture_output=True, text=True, env=env)


def test_parser_defaults_match_reference():
    a = build_parser().parse_args(["train", "-train", "c.txt", "-output", "v.txt"])
    assert (a.size, a.window, a.negative, a.sample, a.min_count, a.alpha, a.iter, a.batch_size) == \
        (300, 5, 5, 1e-4, 5, 0.025, 5, 16)
    d = build_parser().parse_args(["train-dist", "-train", "c", "-output", "v"])
    assert d.sync_period == 1_000_000 and d.hot_rows is None


def test_usage_and_data_errors(tmp_path):
    assert _run("train").returncode == 2
    assert _run("train", "-train", "x", "-output", "y", "-kernel", "scalar").returncode == 2
    assert main(["eval", "-model", str(tmp_path / "missing.vec"), "-similarity", "p"]) == 1
    assert _run("train-dist", "-train", "x", "-output", "y", "-inprocess", "2").returncode == 2


def test_eval_similarity_on_host(tmp_path, capsys):
    from paper_1604_04661_b200.corpus import Vocabulary
    from paper_1604_04661_b200.model import EmbeddingModel, save_model
    rng = np.random.default_rng(0)
    vecs = rng.normal(size=(10, 4)).astype(np.float32)
    toks = [f"t{i}" for i in range(10)]
    voc = Vocabulary(toks, np.ones(10, np.int64), {t: i for i, t in enumerate(toks)}, 10)
    save_model(EmbeddingModel(vecs, np.zeros_like(vecs)), voc, str(tmp_path / "m.vec"))
    (tmp_path / "p.txt").write_text("t1 t2 3\nt3 t4 5\nt0 t9 1\nt5 zz 2\n")
    assert main(["eval", "-model", str(tmp_path / "m.vec"), "-similarity", str(tmp_path / "p.txt")]) == 0
    out = capsys.readouterr().out
    assert "pairs_used: 3" in out and "pairs_skipped: 1" in out


@pytest.mark.gpu
def test_cli_train_writes_vectors_and_report(tmp_path):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("needs CUDA")
    from paper_1604_04661_b200.synthetic import make_planted_corpus
    syn = make_planted_corpus(60_000, 500, n_clusters=4, cluster_size=6, seed=2)
    corpus = tmp_path / "c.txt"
    syn.write_text(str(corpus))
    out, rep = tmp_path / "v.bin", tmp_path / "r.txt"
    r = _run("train", "-train", str(corpus), "-output", str(out), "-size", "32", "-iter", "2",
             "-min-count", "1", "-binary", "1", "-report", str(rep))
    assert r.returncode == 0, r.stderr
    items = dict(line.split(": ", 1) for line in rep.read_text().splitlines())
    assert int(items["words_read"]) == 2 * syn.encoded.n_tokens
    assert items["command"] == "train" and "loss_epoch_2" in items
    from paper_1604_04661_b200.model import load_model
    m, v = load_model(str(out))
    assert m.input_vectors.shape == (syn.vocab.size, 32) and np.isfinite(m.input_vectors).all()


@pytest.mark.gpu
def test_cli_train_dist_under_torchrun(tmp_path):
    """train-dist through torchrun (one process per GPU, NCCL, rendezvous on 127.0.0.1):
    a world of one rank trains, writes the vectors and the rank-0 report."""
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("needs CUDA")
    import socket
    from paper_1604_04661_b200.synthetic import make_planted_corpus
    syn = make_planted_corpus(40_000, 400, n_clusters=4, cluster_size=6, seed=5)
    corpus = tmp_path / "c.txt"
    syn.write_text(str(corpus))
    out, rep = tmp_path / "v.txt", tmp_path / "r.txt"
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=1",
                        "--master-addr", "127.0.0.1", "--master-port", str(port),
                        "-m", "paper_1604_04661_b200", "train-dist", "-train", str(corpus),
                        "-output", str(out), "-size", "16", "-iter", "2", "-min-count", "1",
                        "-sync-period", "20000", "-report", str(rep)],
                       cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    items = dict(line.split(": ", 1) for line in rep.read_text().splitlines())
    assert items["command"] == "train-dist" and items["transport"] == "nccl" and items["nodes"] == "1"
    assert int(items["words_read"]) == 2 * syn.encoded.n_tokens
    from paper_1604_04661_b200.model import load_model
    m, v = load_model(str(out))
    assert m.input_vectors.shape == (syn.vocab.size, 16) and np.isfinite(m.input_vectors).all()
