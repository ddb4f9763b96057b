"""Calibration of the CPU baseline: the oracle port (oracle/, what bench.py's cpu_baseline
and --impl reference arm time on the GPU box) against the real reference package
(numba + OpenBLAS, /root/reference/pkg/src) on the same corpus, config and host cores.

The reference is imported from /root/reference/pkg/src in the build container and from
baseline/_ref (its unmodified pip install, git-ignored, travels with gpurun) on the GPU box:

    OPENBLAS_NUM_THREADS=1 python tools/calibrate_port.py > profiles/round2_port_calibration_gpubox.json

The port runs twice, with its batch_core_naive restatement (bit-exact pins) and its
batch_core_blas restatement (the reference's default float32 backend; bench.py's CPU
baseline).  All sides train one epoch of a seeded 3M-token Zipf(1.05) corpus over 71k ids (configs[2]'s
vocabulary shape), d=300, w=5, K=5, t=1e-4, float32, batch_cap 16, with T = all host
threads (Hogwild), after a warm-up run that JIT-compiles the reference; the metric is the
reference's own (kept words / wall seconds, trainer.py:529-532).
"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
REF_SRC = "/root/reference/pkg/src"
if not os.path.isdir(REF_SRC):
    REF_SRC = os.path.join(ROOT, "baseline", "_ref")  # pip install --target of the same package
sys.path.insert(0, REF_SRC)


def main(tokens=3_000_000, dim=300, seed=1):
    os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
    from sgns import corpus as rc, trainer as rt  # the reference
    from oracle import oracle as O
    from paper_1604_04661_b200.corpus import default_table_length, keep_probabilities
    from paper_1604_04661_b200.model import SIGMOID_TABLE_F32
    from paper_1604_04661_b200.synthetic import make_planted_corpus

    T = len(os.sched_getaffinity(0))
    syn = make_planted_corpus(tokens, 71_000, zipf_s=1.05, min_count=5, seed=0)
    v, e = syn.vocab, syn.encoded
    voc = rc.Vocabulary(list(v.tokens), v.counts.copy(), dict(v.index), int(v.total_tokens))
    enc = rc.EncodedCorpus(e.ids.copy(), e.offsets.copy(), e.sentence_bytes.copy())
    cfg = rt.TrainingConfig(dim=dim, window=5, negatives=5, subsample=1e-4, min_count=5,
                            epochs=1, threads=T, seed=seed)
    # warm-up (numba JIT) on a small slice
    small = rc.EncodedCorpus(enc.ids[:enc.offsets[200]].copy(), enc.offsets[:201].copy(),
                             enc.sentence_bytes[:200].copy())
    rt.train_encoded(voc, small, cfg)
    _, st = rt.train_encoded(voc, enc, cfg)
    ref = {"words_per_sec": st.throughput_words_per_sec, "wall_s": st.wall_seconds,
           "words_trained": st.words_processed, "loss": st.loss_by_epoch[0]}

    counts = v.counts
    V = len(counts)
    keep = keep_probabilities(counts, int(v.total_tokens), 1e-4)
    L = default_table_length(V)
    slots = np.repeat(np.arange(V, dtype=np.int32), np.diff(O.neg_boundaries(counts, 0.75, L), prepend=0))
    ports = {}
    for mm in ("naive", "blas"):
        m_in = O.init_model(V, dim, seed).astype(np.float32)
        m_out = np.zeros((V, dim), np.float32)
        run = O.OracleRun(e.ids, e.offsets.astype(np.int64), m_in, m_out, keep_probs=keep, window=5,
                          negatives=5, batch_cap=16, dynamic=True, seed=seed, alpha0=0.025,
                          floor_frac=1e-4, total_x_epochs=float(e.n_tokens), epochs=1,
                          loss_every=100, n_workers=T, slots=slots, sig_table=SIGMOID_TABLE_F32,
                          refresh_words=10_000, matmul=mm)
        t0 = time.perf_counter()
        while not run.done:
            run.advance(1 << 40, T)
        wall = time.perf_counter() - t0
        trained = sum(w.words_trained for w in run.workers)
        ports[mm] = {"words_per_sec": trained / wall, "wall_s": wall, "words_trained": trained,
                     "loss": float(run.loss.sum() / max(run.cells.sum(), 1)),
                     "over_reference": trained / wall / ref["words_per_sec"]}
    print(json.dumps({
        "what": "oracle port (naive and blas cores) vs the reference package (its default float32 "
                "backend, blas), same corpus/config/cores",
        "host": os.uname().nodename, "reference_from": REF_SRC,
        "corpus": f"{e.n_tokens} tokens Zipf(1.05) over {V} ids (planted clusters), d={dim} w=5 K=5 "
                  "t=1e-4, 1 epoch, float32",
        "threads": T, "cpu": _cpu_model(), "openblas_threads": os.environ.get("OPENBLAS_NUM_THREADS"),
        "reference": ref, "port_naive": ports["naive"], "port_blas": ports["blas"],
    }))


def _cpu_model():
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


if __name__ == "__main__":
    main()
