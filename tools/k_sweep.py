"""Production-path throughput vs the number of negatives K on the configs[2]-shaped corpus
(17M tokens Zipf(1.05) over 71k ids, d=300, w=5, t=1e-4, 2 epochs) through train_encoded.

    python tools/k_sweep.py 5 7 10 15            # schedule "auto" (dynamic where eligible)
    python tools/k_sweep.py --both 10 15         # also the static schedule, for comparison
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main(ks, schedules=("auto",)):
    import paper_1604_04661_b200 as P
    from paper_1604_04661_b200.synthetic import make_planted_corpus
    syn = make_planted_corpus(17_000_000, 71_000, zipf_s=1.05, min_count=5, seed=0)
    for k in ks:
        for sch in schedules:
            cfg = P.TrainingConfig(dim=300, window=5, negatives=k, subsample=1e-4, min_count=5, epochs=2,
                                   seed=1, schedule=sch)
            _, st = P.train_encoded(syn.vocab, syn.encoded, cfg)
            print(json.dumps({"K": k, "schedule": sch, "words_per_sec": st.throughput_words_per_sec,
                              "loss_by_epoch": st.loss_by_epoch}), flush=True)


if __name__ == "__main__":
    args = sys.argv[1:]
    both = "--both" in args
    ks = [int(x) for x in args if x != "--both"] or [5, 7, 10, 15]
    main(ks, ("auto", "static") if both else ("auto",))
