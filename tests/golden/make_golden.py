"""Generate the golden fixtures by running the REFERENCE package in this container.

Usage (from the repo root, only where /root/reference exists):

    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_golden.py

Every array written here is produced by the reference's own functions
(`sgns.*` imported from /root/reference/pkg/src); the synthetic inputs come
from this repo's seeded generator so the same arrays can be rebuilt on the GPU
box, where the reference does not exist.  The fixtures pin the C oracle
(`oracle/`) and, through it, the CUDA path.
"""

from __future__ import annotations

import os
import sys
import threading

import numpy as np

REF_SRC = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REF_SRC)
sys.path.insert(0, ROOT)
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")

import sgns  # noqa: E402  (the reference)
from sgns import corpus as rc, kernel_batched as rk, model as rm, rng as rr  # noqa: E402
from sgns import trainer as rt, distributed as rd, evaluate as rev  # noqa: E402

from paper_1604_04661_b200.synthetic import make_planted_corpus  # noqa: E402

sys.path.insert(0, os.path.dirname(HERE))
from helpers import TRACE_CASES, TRAIN_BASE, TRAIN_CASES  # noqa: E402  (shared with the tests)


def ref_vocab(syn):
    v = syn.vocab
    return rc.Vocabulary(list(v.tokens), v.counts.copy(), dict(v.index), int(v.total_tokens))


def ref_encoded(syn):
    e = syn.encoded
    return rc.EncodedCorpus(e.ids.copy(), e.offsets.copy(), e.sentence_bytes.copy())


def gen_rng():
    out = {}
    cases = [(0, 0), (1, 0), (1, 1), (7, 3), (123456789, 0x1017), (2**63 + 5, 12)]
    for i, (seed, stream) in enumerate(cases):
        st = rr.new_state(seed, stream)
        out[f"c{i}_seed"] = np.array([seed], dtype=np.uint64)
        out[f"c{i}_stream"] = np.array([stream], dtype=np.uint64)
        out[f"c{i}_state0"] = st.copy()
        out[f"c{i}_u64"] = np.array([rr.next_u64(st) for _ in range(64)], dtype=np.uint64)
        out[f"c{i}_uniform"] = np.array([rr.next_uniform(st) for _ in range(64)])
        out[f"c{i}_below7"] = np.array([rr.next_below(st, 7) for _ in range(64)], dtype=np.int64)
        out[f"c{i}_below1e8"] = np.array([rr.next_below(st, 100_000_000) for _ in range(64)], dtype=np.int64)
    out["n_cases"] = np.array([len(cases)])
    np.savez_compressed(os.path.join(HERE, "rng.npz"), **out)


def gen_tables():
    out = {"sigmoid_f32": rm.SIGMOID_TABLE_F32, "sigmoid_f64": rm.SIGMOID_TABLE_F64}
    # probe the float64 bin-index rule around every bin edge (survey App. A)
    edges = -6.0 + np.arange(1000) * (12.0 / 1000)
    probes = []
    for e in edges:
        f = np.float32(e)
        probes += [f, np.nextafter(f, np.float32(-10)), np.nextafter(f, np.float32(10))]
    probes += [np.float32(x) for x in (-100.0, -6.0, -5.99, 0.0, 5.99, 6.0, 7.0, 100.0)]
    probes = np.array(probes, dtype=np.float32)
    out["probe_x"] = probes
    out["probe_sig"] = np.array([rm.sigmoid_from_table(x, rm.SIGMOID_TABLE_F32) for x in probes],
                                dtype=np.float32)
    rng = np.random.default_rng(5)
    counts = np.sort(rng.integers(1, 50_000, size=257))[::-1].astype(np.int64)
    toks = [f"w{i}" for i in range(len(counts))]
    voc = rc.Vocabulary(toks, counts, {t: i for i, t in enumerate(toks)}, int(counts.sum()))
    out["kp_counts"] = counts
    for t in (1e-3, 1e-4, 1e-5):
        out[f"kp_{t:g}"] = voc.keep_probs(t)
    tab = rc.build_negative_table(voc, length=100_003)
    out["neg_small_slots"] = tab.slots
    big_counts = np.sort(rng.integers(1, 2_000_000, size=12_000))[::-1].astype(np.int64)
    toks = [f"w{i}" for i in range(len(big_counts))]
    big = rc.Vocabulary(toks, big_counts, {t: i for i, t in enumerate(toks)}, int(big_counts.sum()))
    btab = rc.build_negative_table(big)  # default 10^8 slots
    out["neg_big_counts"] = big_counts
    out["neg_big_slot_counts"] = np.bincount(btab.slots, minlength=big.size).astype(np.int64)
    for V in (1, 9_999, 10_000, 250_000):
        out[f"deflen_{V}"] = np.array([rc.default_table_length(V)])
    np.savez_compressed(os.path.join(HERE, "tables.npz"), **out)


def gen_init():
    out = {}
    for (V, D, seed) in ((37, 11, 5), (20, 300, 1), (5, 3, 2**40 + 1)):
        m32 = rm.init_model(V, D, seed, dtype=np.float32)
        m64 = rm.init_model(V, D, seed, dtype=np.float64)
        out[f"in32_{V}_{D}_{seed}"] = m32.input_vectors
        out[f"in64_{V}_{D}_{seed}"] = m64.input_vectors
    np.savez_compressed(os.path.join(HERE, "init.npz"), **out)


def make_model(v, d, seed, dtype, scale=1.0):
    rng = np.random.default_rng(seed)
    return rm.EmbeddingModel(rng.normal(scale=scale, size=(v, d)).astype(dtype),
                             rng.normal(scale=scale, size=(v, d)).astype(dtype))


def gen_kernel():
    """process_batch on fixed models: (V, D, in_ids, out_ids, alpha) cases."""
    out = {}
    rng = np.random.default_rng(99)
    cases = [
        (15, 7, [2, 5, 2, 9], [1, 3, 4, 3], 0.07, 1.0),          # dup inputs + dup negative
        (6, 4, [3, 3], [0, 1], 0.1, 1.0),
        (5, 3, [1, 2], [0, 3, 4], 0.0, 1.0),                      # alpha = 0
        (12, 9, [1, 2, 3, 1], [0, 5, 6, 7], 0.05, 1.0),
        (50, 8, [7], [3, 1, 2, 4], 0.05, 0.5),                    # batch cap 1
    ]
    for _ in range(6):  # north-star shapes: d=300/100, m<=10, K=5
        V, D = 32, int(rng.choice([100, 300]))
        m = int(rng.integers(1, 11))
        tgt = int(rng.integers(V))
        negs = [int(x) for x in rng.choice([w for w in range(V) if w != tgt], 5)]
        cases.append((V, D, [int(x) for x in rng.integers(0, V, m)], [tgt] + negs,
                      float(rng.uniform(0.001, 0.05)), float(D) ** -0.25))
    for K in (10, 15):  # microbench K, w=10 full windows (batch_cap >= 20)
        V, D = 40, 200
        tgt = int(rng.integers(V))
        negs = [int(x) for x in rng.choice([w for w in range(V) if w != tgt], K)]
        cases.append((V, D, [int(x) for x in rng.integers(0, V, 20)], [tgt] + negs, 0.025,
                      float(D) ** -0.25))
    out["n_cases"] = np.array([len(cases)])
    for i, (V, D, ins, outs, alpha, scale) in enumerate(cases):
        out[f"c{i}_in_ids"] = np.array(ins, dtype=np.int32)
        out[f"c{i}_out_ids"] = np.array(outs, dtype=np.int32)
        out[f"c{i}_alpha"] = np.array([alpha])
        # f32 base == f64 base cast (make_model draws in f64 then casts), so store f64 only;
        # results are stored for the touched rows only (locality is checked separately)
        rows_in = np.unique(np.array(ins))
        rows_out = np.unique(np.array(outs))
        out[f"c{i}_rows_in"] = rows_in
        out[f"c{i}_rows_out"] = rows_out
        for dt, name in ((np.float32, "f32"), (np.float64, "f64")):
            base = make_model(V, D, 1000 + i, dt, scale)
            if dt == np.float64:
                out[f"c{i}_min"] = base.input_vectors.copy()
                out[f"c{i}_mout"] = base.output_vectors.copy()
            for be in ("blas", "naive"):
                mdl = base.copy()
                rk.process_batch(mdl, rk.Minibatch(np.array(ins), np.array(outs)), alpha, matmul=be)
                untouched_in = np.setdiff1d(np.arange(V), rows_in)
                untouched_out = np.setdiff1d(np.arange(V), rows_out)
                assert np.array_equal(mdl.input_vectors[untouched_in], base.input_vectors[untouched_in])
                assert np.array_equal(mdl.output_vectors[untouched_out], base.output_vectors[untouched_out])
                out[f"c{i}_{name}_{be}_min"] = mdl.input_vectors[rows_in]
                out[f"c{i}_{name}_{be}_mout"] = mdl.output_vectors[rows_out]
    np.savez_compressed(os.path.join(HERE, "kernel.npz"), **out)


def trace_pipeline(vocab, encoded, window, k, cap, dynamic, subsample, seed, stream, table_len):
    """The reference's draw stream as the fused driver consumes it (test_trainer.py:93-138)."""
    table = rc.build_negative_table(vocab, length=table_len)
    keep = vocab.keep_probs(subsample) if subsample > 0 else None
    state = rr.new_state(seed, stream)
    targets, in_off, in_ids, outs, sent_of = [], [0], [], [], []
    for s in range(encoded.n_sentences):
        sent = encoded.sentence(s)
        if keep is not None:
            sent = rc.subsample_sentence(sent, keep, state)
        for b in rk.assemble_batches(rc.iterate_windows(sent, window, state, dynamic),
                                     cap, k, table, state):
            targets.append(int(b.output_ids[0]))
            in_ids.extend(b.input_ids.tolist())
            in_off.append(len(in_ids))
            outs.append(b.output_ids.copy())
            sent_of.append(s)
    return dict(target=np.array(targets, dtype=np.int32), in_off=np.array(in_off, dtype=np.int64),
                in_ids=np.array(in_ids, dtype=np.int32), out_ids=np.array(outs, dtype=np.int32),
                sentence=np.array(sent_of, dtype=np.int64), final_state=state.copy())


def gen_traces():
    out = {}
    for (name, n, V, w, k, cap, dyn, sub, seed, stream, tl) in TRACE_CASES:
        syn = make_planted_corpus(n, V, n_clusters=2, cluster_size=5, sentence_len=37,
                                  seed=int(name[1:]) + 100)
        voc, enc = ref_vocab(syn), ref_encoded(syn)
        tr = trace_pipeline(voc, enc, w, k, cap, dyn, sub, seed, stream, tl)
        out[f"{name}_ids"] = enc.ids
        out[f"{name}_offsets"] = enc.offsets
        out[f"{name}_counts"] = voc.counts
        for key, val in tr.items():
            out[f"{name}_{key}"] = val
    np.savez_compressed(os.path.join(HERE, "traces.npz"), **out)


def train_corpus():
    return make_planted_corpus(30_000, 300, n_clusters=5, cluster_size=6, sentence_len=50, seed=42)


def gen_train():
    syn = train_corpus()
    voc, enc = ref_vocab(syn), ref_encoded(syn)
    out = {"ids": enc.ids, "offsets": enc.offsets, "counts": voc.counts,
           "sentence_bytes": enc.sentence_bytes}
    for name, kw in TRAIN_CASES.items():
        base = dict(TRAIN_BASE)
        base.update(kw)
        cfg = rt.TrainingConfig(**base)
        model, stats = rt.train_encoded(voc, enc, cfg)
        out[f"{name}_min"] = model.input_vectors
        out[f"{name}_mout"] = model.output_vectors
        out[f"{name}_stats"] = np.array([stats.words_processed, stats.words_read], dtype=np.int64)
        out[f"{name}_final_alpha"] = np.array([stats.final_alpha])
        out[f"{name}_loss"] = np.array(stats.loss_by_epoch)
    np.savez_compressed(os.path.join(HERE, "train.npz"), **out)


def gen_dist():
    out = {}
    k = 0
    for V in (1, 50, 10_000, 10_001, 123_457):
        for pol in (rd.SyncPolicy(), rd.SyncPolicy(hot_rows=3, rotation_chunk=2),
                    rd.SyncPolicy(hot_rows=0), rd.SyncPolicy(hot_rows=V, rotation_chunk=0)):
            if pol.hot_rows is not None and pol.hot_rows > V:
                continue
            for period in (0, 1, 19, 20, 57):
                rows = rd.select_sync_rows(V, pol, period)
                # stored as [lo, hi) runs; the tests expand them
                brk = np.flatnonzero(np.diff(rows) != 1) + 1 if len(rows) else np.array([], int)
                starts = np.concatenate([[0], brk]) if len(rows) else np.array([], int)
                stops = np.concatenate([brk, [len(rows)]]) if len(rows) else np.array([], int)
                runs = np.array([[rows[a], rows[b - 1] + 1] for a, b in zip(starts, stops)],
                                dtype=np.int64).reshape(-1, 2)
                out[f"s{k}_args"] = np.array([V, -1 if pol.hot_rows is None else pol.hot_rows,
                                              -1 if pol.rotation_chunk is None else pol.rotation_chunk,
                                              period], dtype=np.int64)
                out[f"s{k}_runs"] = runs
                out[f"s{k}_len"] = np.array([len(rows)])
                k += 1
    out["n_sync"] = np.array([k])
    syn = train_corpus()
    enc = ref_encoded(syn)
    for n in (1, 2, 3, 8):
        out[f"part_{n}"] = np.array(rc.partition_sentences(enc, n), dtype=np.int64)
        out[f"split_{n}"] = np.array(rt.split_by_tokens(enc.offsets, 0, enc.n_sentences, n), dtype=np.int64)
        lo, hi = rc.partition_sentences(enc, 2)[1]
        out[f"split_sub_{n}"] = np.array(rt.split_by_tokens(enc.offsets, lo, hi, n), dtype=np.int64)
    out["split_big"] = np.array(rt.split_by_tokens(enc.offsets, 0, enc.n_sentences, 700), dtype=np.int64)
    # in-process N=2 data-parallel run (float64, deterministic: rank-order f64 mean)
    group = rd.InProcessGroup(2)
    res = [None, None]
    cfg = rt.TrainingConfig(dim=8, window=3, negatives=3, subsample=1e-3, min_count=1,
                            epochs=2, threads=1, seed=4, float64=True)
    pol = rd.SyncPolicy(period_words=4000, hot_rows=20, rotation_chunk=30)
    voc = ref_vocab(syn)

    def work(r, ep):
        res[r] = rd.distributed_train(None, cfg, pol, ep, prebuilt=(voc, enc))

    ths = [threading.Thread(target=work, args=(r, ep)) for r, ep in enumerate(group.endpoints())]
    [t.start() for t in ths]
    [t.join() for t in ths]
    out["dp2_min"] = res[0][0].input_vectors
    out["dp2_mout"] = res[0][0].output_vectors
    out["dp2_stats"] = np.array([res[0][1].words_processed, res[0][1].words_read,
                                 res[1][1].words_processed, res[1][1].words_read], dtype=np.int64)
    out["dp2_loss0"] = np.array(res[0][1].loss_by_epoch)
    np.savez_compressed(os.path.join(HERE, "dist.npz"), **out)


def gen_eval_full():
    """eval_similarity / eval_analogy of the reference on random vectors, header lines,
    OOV words, lowercase fallback, sections and max_vocab."""
    rng = np.random.default_rng(12)
    V, D = 400, 24
    toks = [f"w{i}" for i in range(V - 2)] + ["Paris", "rome"]
    voc = rc.Vocabulary(toks, np.arange(V, 0, -1, dtype=np.int64), {t: i for i, t in enumerate(toks)}, 1)
    vecs = rng.normal(size=(V, D)).astype(np.float32)
    vecs[5] = 0.0  # zero row: analogy normalisation guard
    model = rm.EmbeddingModel(vecs, np.zeros_like(vecs))
    sim = ["word1 word2 score"]
    for _ in range(150):
        a, b = rng.integers(0, V, 2)
        if a == 5 or b == 5:
            continue
        sim.append(f"{toks[a]} {toks[b]} {rng.uniform(0, 10):.2f}")
    sim += ["PARIS Rome 7.5", "oov1 w3 2.0"]
    ana = []
    unit = vecs / np.maximum(np.linalg.norm(vecs, axis=1, keepdims=True), 1e-30)
    for sec in range(4):
        ana.append(f": section{sec}")
        for _ in range(120):
            ids = rng.integers(0, V, 4)
            if rng.random() < 0.7:  # make most answers the true 3CosAdd argmax
                sc = (unit[ids[1]] - unit[ids[0]] + unit[ids[2]]) @ unit.T
                sc[ids[:3]] = -np.inf
                ids[3] = int(np.argmax(sc))
            ana.append(" ".join(toks[i] for i in ids))
        ana.append("w1 w2 oov w3")
    sim_path, ana_path = "/tmp/golden_sim.txt", "/tmp/golden_ana.txt"
    open(sim_path, "w").write("\n".join(sim) + "\n")
    open(ana_path, "w").write("\n".join(ana) + "\n")
    rho, used, skipped = rev.eval_similarity(model, voc, sim_path)
    acc, by_sec, sk = rev.eval_analogy(model, voc, ana_path)
    acc2, by_sec2, sk2 = rev.eval_analogy(model, voc, ana_path, max_vocab=250, block=64)
    np.savez_compressed(os.path.join(HERE, "eval_full.npz"), vecs=vecs, tokens=np.array("\x00".join(toks)),
                        sim=np.array("\n".join(sim) + "\n"), ana=np.array("\n".join(ana) + "\n"),
                        sim_out=np.array([rho, used, skipped]),
                        ana_out=np.array([acc, sk, acc2, sk2]),
                        ana_sec=np.array([[by_sec[f"section{k}"][0], by_sec[f"section{k}"][1],
                                           by_sec2[f"section{k}"][0], by_sec2[f"section{k}"][1]] for k in range(4)]))


def gen_eval():
    syn = make_planted_corpus(20_000, 500, n_clusters=6, cluster_size=8, seed=9)
    voc = ref_vocab(syn)
    pairs = os.path.join("/tmp", "golden_pairs.txt")
    syn.write_gold_pairs(pairs, pairs_per_cluster=10)
    rng = np.random.default_rng(3)
    vecs = rng.normal(size=(voc.size, 12)).astype(np.float32)
    model = rm.EmbeddingModel(vecs, np.zeros_like(vecs))
    rho, used, skipped = rev.eval_similarity(model, voc, pairs)
    with open(pairs) as fh:
        text = fh.read()
    np.savez_compressed(os.path.join(HERE, "eval.npz"), vecs=vecs, counts=voc.counts,
                        pairs=np.array([text]), rho=np.array([rho, used, skipped]))


def gen_ingest():
    """A text corpus exercising every str.split() whitespace class, universal newlines,
    >1000-token lines, OOV-only and empty lines and an unterminated last line; the
    reference's build_vocab(read_tokens) / encode_corpus outputs pin the C++ scanner."""
    rng = np.random.default_rng(77)
    words = [f"w{i}" for i in range(300)] + ["naïve", "日本語", "über", "ça", "x\u200by", "Ω", "a", "A"]
    p = 1.0 / np.arange(1, len(words) + 1)
    p /= p.sum()
    seps = [" ", " ", " ", "\t", "\x0b", "\x0c", "\x1c", "\x1f", "\xa0", "\u2003", "\u3000",
            "\x85", "\u2028", "\u205f", "  \t "]
    ends = ["\n", "\n", "\r\n", "\r"]
    lines = []
    for li in range(400):
        n = int(rng.integers(0, 40)) if li % 50 else int(rng.integers(1000, 2600))
        toks = [words[i] for i in rng.choice(len(words), size=n, p=p)]
        if li % 37 == 5:
            toks = [f"oov{li}_{k}" for k in range(5)]
        body = ""
        for t in toks:
            body += t + seps[int(rng.integers(len(seps)))]
        if li % 9 == 0:
            body = seps[int(rng.integers(len(seps)))] + body
        lines.append(body + ends[int(rng.integers(len(ends)))])
    text = "".join(lines) + "w1 w2 tail"  # unterminated last line
    path = os.path.join(HERE, "ingest_corpus.txt")
    with open(path, "w", encoding="utf-8", newline="") as fh:
        fh.write(text)
    voc = rc.build_vocab(rc.read_tokens(path), 2)
    enc = rc.encode_corpus(path, voc)
    np.savez_compressed(os.path.join(HERE, "ingest.npz"),
                        tokens=np.array("\x00".join(voc.tokens)), counts=voc.counts,
                        total=np.array([voc.total_tokens]), ids=enc.ids, offsets=enc.offsets,
                        sentence_bytes=enc.sentence_bytes)


def gen_io():
    """save_model text and binary bytes from the reference, on values that stress %.6g."""
    rng = np.random.default_rng(31)
    V, D = 23, 7
    vecs = (rng.normal(size=(V, D)) * 10.0 ** rng.integers(-9, 9, size=(V, D))).astype(np.float32)
    vecs[0, :] = [0.0, -0.0, 1e-45, 3.4e38, 123456.5, 1234567.0, 0.1]
    toks = [f"w{i}" for i in range(V - 2)] + ["naïve", "日本語"]
    voc = rc.Vocabulary(toks, np.arange(V, 0, -1, dtype=np.int64), {t: i for i, t in enumerate(toks)},
                        int(np.arange(V, 0, -1).sum()))
    model = rm.EmbeddingModel(vecs, np.zeros_like(vecs))
    out = {"vecs": vecs, "tokens": np.array("\x00".join(toks))}
    for binary in (False, True):
        path = os.path.join("/tmp", f"golden_vec_{int(binary)}")
        rm.save_model(model, voc, path, binary=binary)
        with open(path, "rb") as fh:
            out[f"bytes_{int(binary)}"] = np.frombuffer(fh.read(), dtype=np.uint8)
    # float64 model: the reference formats the float64 value itself (%.6g); values sit next
    # to a 6th-digit rounding boundary, where a float32 cast would print differently
    v64 = rng.normal(size=(V, D)) * 10.0 ** rng.integers(-5, 5, size=(V, D))
    v64[1, :] = [1.2345650000000001, 1.2345649999999999, 0.30000000000000004, 2.5e-300,
                 9.9999995e-5, 123456.49999999999, -7.77777750000001]
    out["vecs64"] = v64
    model64 = rm.EmbeddingModel(v64, np.zeros_like(v64))
    for binary in (False, True):
        path = os.path.join("/tmp", f"golden_vec64_{int(binary)}")
        rm.save_model(model64, voc, path, binary=binary)
        with open(path, "rb") as fh:
            out[f"bytes64_{int(binary)}"] = np.frombuffer(fh.read(), dtype=np.uint8)
    np.savez_compressed(os.path.join(HERE, "io.npz"), **out)


READ_CASES = [
    # (name, file bytes, binary flag passed to load_model: None = detect_format)
    ("plain", b"3 2\na 1 2\nb -0.5 3e-3\nc 1e10 -7\n", None),
    ("py_numbers", b"3 3\nx +1.5 1_000.25 .5\ny 5. -.25e+2 1E-45\nz inf -Infinity nan\n", None),
    ("crlf_and_cr", b"2 2\r\na 1 2\r\nb 3 4\rc 9 9\n", False),
    ("tab_in_field", b"2 2\na \t1 2\nb 3 4\t\n", False),
    ("fullwidth_digits", "2 2\nu \uff11.5 2\nv 3 \u0664\n".encode(), False),
    ("utf8_tokens", "2 2\nnaïve 1 2\n日本語 3 4\n".encode(), None),
    ("no_final_newline", b"2 2\na 1 2\nb 3 4", None),
    ("dup_tokens", b"3 1\na 1\nb 2\na 3\n", None),
    ("extra_field", b"2 2\na 1 2\nb 3 4 5\n", False),
    ("missing_field", b"2 2\na 1\nb 3 4\n", False),
    ("blank_line", b"2 2\na 1 2\n\nb 3 4\n", False),
    ("double_space", b"2 2\na 1  2\nb 3 4\n", False),
    ("bad_number", b"2 2\na 1 2\nb 3 x4\n", False),
    ("truncated_text", b"3 2\na 1 2\nb 3 4\n", False),
    ("bad_header", b"3 x\na 1 2\n", None),
    ("header_three", b"3 2 1\na 1 2\n", None),
    ("header_zero", b"0 2\n", None),
    ("header_underscore", b"1_0 1\n" + b"".join(b"w%d %d\n" % (i, i) for i in range(10)), None),
    ("bin_plain", b"2 2\n" + b"a " + np.array([1.5, -2], "<f4").tobytes() + b"\n" + b"bb "
     + np.array([3, 4], "<f4").tobytes() + b"\n", None),
    ("bin_no_newlines", b"2 1\n" + b"a " + np.array([1], "<f4").tobytes() + b"b "
     + np.array([2], "<f4").tobytes(), True),
    ("bin_leading_newline_token", b"2 1\n\na " + np.array([1], "<f4").tobytes() + b"\n\n\nb "
     + np.array([2], "<f4").tobytes(), True),
    ("bin_truncated_payload", b"2 2\na " + np.array([1, 2], "<f4").tobytes() + b"\nb \x00\x00", True),
    ("bin_truncated_token", b"2 2\na " + np.array([1, 2], "<f4").tobytes() + b"\nbbb", True),
    ("bin_bad_utf8", b"1 1\n\xff\xfe " + np.array([1], "<f4").tobytes() + b"\n", True),
    ("bin_space_payload", b"2 1\n" + b"a " + np.array([np.float32(32.0 / 2 ** 126)], "<f4").tobytes()
     + b"\nb " + np.array([8.0], "<f4").tobytes() + b"\n", True),
    ("sniff_binary", b"2 2\n" + b"a " + np.array([1e-3, 7], "<f4").tobytes() + b"\nb "
     + np.array([3, 4], "<f4").tobytes() + b"\n", None),
    ("sniff_short_text", b"4 3\na 1\n", None),
    ("sniff_empty_body", b"2 2\n", None),
    ("text_bad_utf8", b"2 1\na 1\n\xc3 2\n", False),
]


def gen_read():
    """The reference's load_model (and detect_format) outcome on every READ_CASES file:
    tokens and float32 bits, or the exception class and message."""
    out = {"names": np.array("\x00".join(c[0] for c in READ_CASES))}
    for name, data, binary in READ_CASES:
        path = os.path.join("/tmp", "golden_read_" + name)
        with open(path, "wb") as fh:
            fh.write(data)
        out[f"{name}__bytes"] = np.frombuffer(data, dtype=np.uint8)
        out[f"{name}__binary"] = np.array(-1 if binary is None else int(binary))
        try:
            model, voc = rm.load_model(path, binary)
            out[f"{name}__tokens"] = np.array("\x00".join(voc.tokens))
            out[f"{name}__vecs"] = model.input_vectors.view(np.uint32)
        except Exception as exc:  # noqa: BLE001 -- the outcome is the fixture
            out[f"{name}__error"] = np.array(type(exc).__name__ + ": " + str(exc).replace(path, "<path>"))
        try:
            out[f"{name}__sniff"] = np.array(int(rm.detect_format(path)))
        except Exception as exc:  # noqa: BLE001
            out[f"{name}__sniff_error"] = np.array(type(exc).__name__)
    np.savez_compressed(os.path.join(HERE, "read.npz"), **out)


if __name__ == "__main__":
    assert sgns.__version__
    only = set(sys.argv[1:])  # e.g. "gen_io": regenerate one fixture
    for fn in (gen_rng, gen_tables, gen_init, gen_kernel, gen_traces, gen_train, gen_dist, gen_eval,
               gen_ingest, gen_io, gen_eval_full, gen_read):
        if only and fn.__name__ not in only:
            continue
        fn()
        print("wrote", fn.__name__)
