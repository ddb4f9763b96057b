"""BASELINE.json configs[2] end to end: 17M-token Zipf(1.05) corpus over 71k ids with
planted clusters, d=300, w=5, K=5, t=1e-4, 5 epochs -- one B200 (production path)
against the reference algorithm on all host cores (the oracle, test infrastructure).

Prints one JSON report: throughput of both, per-epoch loss (every cell scored on both
sides), planted-cluster Spearman rho (mean of the seeds).  Run on the GPU box:

    python tools/run_mid.py [--seeds 1] [--epochs 5] > profiles/round1_mid.json
"""

import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--seeds", type=int, default=1)
    ap.add_argument("--epochs", type=int, default=5)
    ap.add_argument("--tokens", type=int, default=17_000_000)
    ap.add_argument("--vocab", type=int, default=71_000,
                    help="raw ids (configs[2]: 71k; configs[3]: 1M with --tokens 800M --epochs 1)")
    ap.add_argument("--skip-cpu", action="store_true")
    ap.add_argument("--gpu-rng", choices=["philox", "splitmix"], default="philox",
                    help="splitmix: the reference's stream + 1e8-slot table on the GPU (static schedule)")
    ap.add_argument("--gpu-workers", type=int, default=0, help="0: the config default")
    args = ap.parse_args()
    import paper_1604_04661_b200 as P
    from oracle import oracle as O
    from paper_1604_04661_b200.corpus import default_table_length, keep_probabilities
    from paper_1604_04661_b200.evaluate import similarity_score
    from paper_1604_04661_b200.model import SIGMOID_TABLE_F32
    from paper_1604_04661_b200.synthetic import make_planted_corpus

    t0 = time.perf_counter()
    syn = make_planted_corpus(args.tokens, args.vocab, zipf_s=1.05, min_count=5, seed=0)
    gen = time.perf_counter() - t0
    pairs = syn.gold_pairs(pairs_per_cluster=16)
    counts = syn.vocab.counts
    V, D = len(counts), 300
    T = len(os.sched_getaffinity(0))
    report = {"config": f"{args.tokens:,} tokens Zipf(1.05) over {args.vocab:,} raw ids, planted clusters, "
                        f"min-count 5, d=300 w=5 K=5 t=1e-4, {args.epochs} epochs "
                        "(configs[2]: 17M / 71k / 5 epochs; configs[3]: 800M / 1M / 1 epoch)", "vocab": V,
              "tokens": syn.encoded.n_tokens, "corpus_gen_s": gen, "host_cores": T, "runs": []}
    for seed in range(1, args.seeds + 1):
        cfg = P.TrainingConfig(dim=D, window=5, negatives=5, subsample=1e-4, min_count=5, alpha0=0.025,
                               epochs=args.epochs, seed=seed, loss_sample_every=1, rng=args.gpu_rng,
                               workers=args.gpu_workers or None)
        model, st = P.train_encoded(syn.vocab, syn.encoded, cfg)
        rho_g = similarity_score(model.input_vectors, syn.vocab.index, pairs)[0] / 100
        run = {"seed": seed, "gpu_rng": args.gpu_rng, "gpu": {"words_per_sec": st.throughput_words_per_sec, "wall_s": st.wall_seconds,
                                     "loss_by_epoch": st.loss_by_epoch, "rho": rho_g,
                                     "words_trained": st.words_processed}}
        if not args.skip_cpu:
            L = default_table_length(V)
            slots = np.repeat(np.arange(V, dtype=np.int32), np.diff(O.neg_boundaries(counts, 0.75, L), prepend=0))
            m_in = O.init_model(V, D, seed).astype(np.float32)
            m_out = np.zeros((V, D), np.float32)
            orc = O.OracleRun(syn.encoded.ids, syn.encoded.offsets, m_in, m_out,
                              keep_probs=keep_probabilities(counts, int(counts.sum()), 1e-4), window=5,
                              negatives=5, batch_cap=16, dynamic=True, seed=seed, alpha0=0.025,
                              floor_frac=1e-4, total_x_epochs=float(syn.encoded.n_tokens) * args.epochs,
                              epochs=args.epochs, loss_every=1, n_workers=T, slots=slots,
                              sig_table=SIGMOID_TABLE_F32, matmul="blas")
            t1 = time.perf_counter()
            orc.run_to_completion(n_threads=T)
            wall = time.perf_counter() - t1
            trained, read, loss = orc.stats()
            rho_c = similarity_score(m_in, syn.vocab.index, pairs)[0] / 100
            run["cpu_reference"] = {"words_per_sec": trained / wall, "wall_s": wall, "threads": T,
                                    "loss_by_epoch": loss, "rho": rho_c, "words_trained": trained}
            run["loss_rel_diff_by_epoch"] = [g / c - 1 for g, c in zip(st.loss_by_epoch, loss)]
            run["rho_diff"] = rho_g - rho_c
            run["speedup"] = st.throughput_words_per_sec / (trained / wall)
        report["runs"].append(run)
        print(json.dumps(run), file=sys.stderr, flush=True)
    print(json.dumps(report, indent=1))


if __name__ == "__main__":
    main()
