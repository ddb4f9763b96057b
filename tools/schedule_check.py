"""Throughput of the static vs the dynamic (fast) driver schedule at a few K on the configs[2]-shaped corpus."""
import sys, json
import os; sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1604_04661_b200 as P
from paper_1604_04661_b200.synthetic import make_planted_corpus
syn = make_planted_corpus(17_000_000, 71_000, zipf_s=1.05, min_count=5, seed=0)
for k, sch in ((5, "static"), (5, "dynamic"), (7, "static"), (7, "dynamic")):
    cfg = P.TrainingConfig(dim=300, window=5, negatives=k, subsample=1e-4, min_count=5, epochs=2, seed=1, schedule=sch)
    _, st = P.train_encoded(syn.vocab, syn.encoded, cfg)
    print(json.dumps({"K": k, "schedule": sch, "words_per_sec": st.throughput_words_per_sec}), flush=True)
