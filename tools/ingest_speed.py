"""Ingestion throughput: native C++ scanner vs the Python restatement (= reference speed)."""
import os
import sys
import tempfile
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1604_04661_b200.corpus import (build_vocab, build_vocab_file, encode_corpus,  # noqa: E402
                                          encode_corpus_file, read_tokens)
from paper_1604_04661_b200.synthetic import make_planted_corpus  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 20_000_000
syn = make_planted_corpus(n, 71_000, zipf_s=1.05, seed=0)
path = os.path.join(tempfile.mkdtemp(), "corpus.txt")
syn.write_text(path)
mb = os.path.getsize(path) / 1e6
t = time.perf_counter(); v = build_vocab_file(path, 5); e = encode_corpus_file(path, v); tn = time.perf_counter() - t
print(f"{n} tokens, {mb:.0f} MB text, {len(os.sched_getaffinity(0))} threads: native {tn:.2f} s "
      f"({n / tn / 1e6:.1f}M tok/s)")
if n <= 20_000_000:
    t = time.perf_counter(); v2 = build_vocab(read_tokens(path), 5); e2 = encode_corpus(path, v2); tp = time.perf_counter() - t
    print(f"python {tp:.2f} s ({n / tp / 1e6:.2f}M tok/s), speedup {tp / tn:.1f}x, identical "
          f"{v.tokens == v2.tokens and (e.ids == e2.ids).all()}")
