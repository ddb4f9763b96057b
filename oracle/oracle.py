"""ctypes front end of the C oracle (TEST INFRASTRUCTURE ONLY).

Loaded by tests/, __graft_entry__.smoke() and bench.py's CPU-baseline leg as
the checker / CPU baseline; the package `paper_1604_04661_b200` never imports
it.  See sgns_oracle.c for the reference file:line map.
"""

from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "liboracle.so")


def build() -> str:
    subprocess.run(["make", "-s", "-C", HERE], check=True)
    return LIB_PATH


def _load() -> C.CDLL:
    src = os.path.join(HERE, "sgns_oracle.c")
    if not os.path.exists(LIB_PATH) or (
            os.path.exists(src) and os.path.getmtime(src) > os.path.getmtime(LIB_PATH)):
        build()
    return C.CDLL(LIB_PATH)


_lib = _load()
P = C.c_void_p
I32, I64, U64, F64 = C.c_int32, C.c_int64, C.c_uint64, C.c_double


class Worker(C.Structure):
    _fields_ = [("next_sent", I64), ("lo", I64), ("hi", I64), ("epoch", I32), ("done", I32),
                ("rng", U64), ("alpha", F64), ("read_local", F64), ("trained_local", F64),
                ("kernel_counter", I64), ("words_read", I64), ("words_trained", I64)]


class Drive(C.Structure):
    _fields_ = [("dtype", C.c_int), ("m_in", P), ("m_out", P), ("ld", I64), ("D", C.c_int),
                ("ids", P), ("offsets", P), ("keep_probs", P), ("rng_mode", C.c_int),
                ("slots", P), ("n_slots", I64), ("alias_thr", P), ("alias_idx", P),
                ("vocab", I64), ("seed", U64),
                ("window", C.c_int), ("dynamic", C.c_int), ("k_neg", C.c_int),
                ("batch_cap", C.c_int), ("use_exact", C.c_int), ("sig_table", P),
                ("alpha0", F64), ("floor_frac", F64), ("total_x_epochs", F64),
                ("refresh_words", I64), ("shared", P), ("epochs", C.c_int),
                ("loss_every", C.c_int), ("workers", P), ("n_workers", C.c_int),
                ("word_budget", I64), ("loss_by_epoch", P), ("cells_by_epoch", P),
                ("update", C.c_int), ("trace_cap", I64), ("trace", P), ("trace_alpha", P),
                ("trace_count", P), ("position_mode", C.c_int), ("matmul", C.c_int)]


assert _lib.or_sizeof_worker() == C.sizeof(Worker)
assert _lib.or_sizeof_drive() == C.sizeof(Drive)

_lib.or_new_state.restype = U64
_lib.or_new_state.argtypes = [U64, U64]
_lib.or_splitmix_u64.argtypes = [P, P, I64]
_lib.or_splitmix_uniform.argtypes = [P, P, I64]
_lib.or_splitmix_below.argtypes = [P, U64, P, I64]
_lib.or_philox4x32_10.argtypes = [P, P, P]
_lib.or_sigmoid_table_f32.restype = C.c_float
_lib.or_sigmoid_table_f32.argtypes = [C.c_float, P]
_lib.or_process_batch.argtypes = [C.c_int, P, P, I64, C.c_int, P, C.c_int, P, C.c_int, F64,
                                  C.c_int, P, C.c_int]
_lib.or_process_windows.argtypes = [C.c_int, P, P, I64, C.c_int, P, P, P, I64, C.c_int, F64,
                                    C.c_int, P, C.c_int, C.c_int]
MATMUL = {"naive": 0, "blas": 1}
_lib.or_init_model.argtypes = [I64, C.c_int, U64, P]
_lib.or_neg_boundaries.argtypes = [P, I64, F64, I64, P]
_lib.or_drive.argtypes = [C.POINTER(Drive), C.c_int]


def _p(a: np.ndarray | None):
    return None if a is None else a.ctypes.data_as(P)


def new_state(seed: int, stream: int = 0) -> int:
    return int(_lib.or_new_state(seed & (2**64 - 1), stream & (2**64 - 1)))


def splitmix(state: int, n: int, kind: str = "u64", bound: int = 0):
    st = np.array([state], dtype=np.uint64)
    if kind == "u64":
        out = np.empty(n, dtype=np.uint64)
        _lib.or_splitmix_u64(_p(st), _p(out), n)
    elif kind == "uniform":
        out = np.empty(n, dtype=np.float64)
        _lib.or_splitmix_uniform(_p(st), _p(out), n)
    else:
        out = np.empty(n, dtype=np.int64)
        _lib.or_splitmix_below(_p(st), bound, _p(out), n)
    return out, int(st[0])


def philox(ctr, key) -> np.ndarray:
    c = np.asarray(ctr, dtype=np.uint32)
    k = np.asarray(key, dtype=np.uint32)
    o = np.empty(4, dtype=np.uint32)
    _lib.or_philox4x32_10(_p(c), _p(k), _p(o))
    return o


def sigmoid_table_f32(x: float, table: np.ndarray) -> np.float32:
    return np.float32(_lib.or_sigmoid_table_f32(float(np.float32(x)), _p(table)))


def process_batch(m_in: np.ndarray, m_out: np.ndarray, in_ids, out_ids, alpha: float,
                  table: np.ndarray, matmul: str = "naive") -> None:
    """batch_core_naive in place (matmul="blas": the float32 batch_core_blas restatement);
    float64 models use the exact sigmoid (as the reference)."""
    assert m_in.flags.c_contiguous and m_out.flags.c_contiguous and m_in.dtype == m_out.dtype
    dtype = 1 if m_in.dtype == np.float64 else 0
    ins = np.ascontiguousarray(in_ids, dtype=np.int32)
    outs = np.ascontiguousarray(out_ids, dtype=np.int32)
    tab = np.ascontiguousarray(table, dtype=m_in.dtype)
    _lib.or_process_batch(dtype, _p(m_in), _p(m_out), m_in.shape[1], m_in.shape[1], _p(ins),
                          len(ins), _p(outs), len(outs), float(alpha), dtype, _p(tab), MATMUL[matmul])


def process_windows(m_in: np.ndarray, m_out: np.ndarray, in_off, in_ids, out_ids, alpha: float,
                    table: np.ndarray, n_threads: int = 1, matmul: str = "naive") -> None:
    """Packed windows in place (out_ids n_win x K1); n_threads Hogwild threads on contiguous
    window ranges; one thread == sequential process_batch calls.  matmul as process_batch."""
    assert m_in.flags.c_contiguous and m_out.flags.c_contiguous and m_in.dtype == m_out.dtype
    dtype = 1 if m_in.dtype == np.float64 else 0
    off = np.ascontiguousarray(in_off, dtype=np.int32)
    ins = np.ascontiguousarray(in_ids, dtype=np.int32)
    outs = np.ascontiguousarray(out_ids, dtype=np.int32)
    tab = np.ascontiguousarray(table, dtype=m_in.dtype)
    n_win = len(off) - 1
    k1 = outs.size // max(n_win, 1)
    assert outs.size == n_win * k1
    if _lib.or_process_windows(dtype, _p(m_in), _p(m_out), m_in.shape[1], m_in.shape[1], _p(off),
                               _p(ins), _p(outs), n_win, k1, float(alpha), dtype, _p(tab),
                               int(n_threads), MATMUL[matmul]) != 0:
        raise MemoryError("or_process_windows")


def init_model(V: int, D: int, seed: int) -> np.ndarray:
    out = np.empty((V, D), dtype=np.float64)
    _lib.or_init_model(V, D, seed & (2**64 - 1), _p(out))
    return out


def neg_boundaries(counts, power: float, length: int) -> np.ndarray:
    c = np.ascontiguousarray(counts, dtype=np.int64)
    out = np.empty(len(c), dtype=np.int64)
    _lib.or_neg_boundaries(_p(c), len(c), power, length, _p(out))
    return out


def split_by_tokens(offsets, lo, hi, parts):
    base = offsets[lo]
    tokens = offsets[lo + 1:hi + 1] - base
    total = float(tokens[-1]) if len(tokens) else 0.0
    bounds = [lo]
    for k in range(1, parts):
        cut = lo + int(np.searchsorted(tokens, total * k / parts)) + 1
        bounds.append(min(max(cut, bounds[-1]), hi))
    bounds.append(hi)
    return [(bounds[i], bounds[i + 1]) for i in range(parts)]


class OracleRun:
    """All workers of one rank; mirrors ThreadRun (trainer.py:332-453) per worker.

    rng_mode "splitmix": reference stream per worker (stream_base + w) and the
    reference slot table; "philox": counter-based stream + alias table (the
    device production sampler, restated for bit-exact trace checks).
    """

    def __init__(self, ids, offsets, m_in, m_out, *, keep_probs, window, negatives, batch_cap,
                 dynamic, seed, alpha0, floor_frac, total_x_epochs, epochs, loss_every,
                 n_workers, sent_range=None, stream_base=0, rng_mode="splitmix", slots=None,
                 alias=None, sig_table=None, refresh_words=10_000, trace_cap=0, update=True,
                 use_exact=None, position_mode=False, matmul="naive"):
        self.ids = np.ascontiguousarray(ids, dtype=np.int32)
        self.offsets = np.ascontiguousarray(offsets, dtype=np.int64)
        self.m_in, self.m_out = m_in, m_out
        assert m_in.flags.c_contiguous and m_out.flags.c_contiguous
        self.keep = None if keep_probs is None else np.ascontiguousarray(keep_probs, np.float64)
        self.sig = np.ascontiguousarray(sig_table, dtype=m_in.dtype)
        self.slots = None if slots is None else np.ascontiguousarray(slots, dtype=np.int32)
        self.alias_thr = self.alias_idx = None
        if alias is not None:
            self.alias_thr = np.ascontiguousarray(alias[0], dtype=np.uint32)
            self.alias_idx = np.ascontiguousarray(alias[1], dtype=np.int32)
        lo, hi = sent_range if sent_range is not None else (0, len(self.offsets) - 1)
        ranges = split_by_tokens(self.offsets, lo, hi, n_workers)
        self.workers = (Worker * n_workers)()
        for w, (a, b) in enumerate(ranges):
            wk = self.workers[w]
            wk.next_sent, wk.lo, wk.hi = a, a, b
            wk.rng = new_state(seed, stream_base + w)
            wk.alpha = alpha0
        self.shared = np.zeros(2, dtype=np.int64)
        self.loss = np.zeros((n_workers, epochs))
        self.cells = np.zeros((n_workers, epochs), dtype=np.int64)
        k1 = negatives + 1
        self.rec_len = 4 + batch_cap + k1
        self.trace_cap = trace_cap
        self.trace = np.zeros((n_workers, max(trace_cap, 1), self.rec_len), dtype=np.int32)
        self.trace_alpha = np.zeros((n_workers, max(trace_cap, 1)))
        self.trace_count = np.zeros(n_workers, dtype=np.int64)
        d = Drive()
        d.dtype = 1 if m_in.dtype == np.float64 else 0
        d.m_in, d.m_out = _p(m_in), _p(m_out)
        d.ld, d.D = m_in.shape[1], m_in.shape[1]
        d.ids, d.offsets, d.keep_probs = _p(self.ids), _p(self.offsets), _p(self.keep)
        d.rng_mode = 1 if rng_mode == "philox" else 0
        d.slots = _p(self.slots)
        d.n_slots = 0 if self.slots is None else len(self.slots)
        d.alias_thr, d.alias_idx = _p(self.alias_thr), _p(self.alias_idx)
        d.vocab = m_in.shape[0]
        d.seed = seed & (2**64 - 1)
        d.window, d.dynamic, d.k_neg, d.batch_cap = window, int(dynamic), negatives, batch_cap
        d.use_exact = d.dtype if use_exact is None else int(use_exact)
        d.sig_table = _p(self.sig)
        d.alpha0, d.floor_frac, d.total_x_epochs = alpha0, floor_frac, total_x_epochs
        d.refresh_words = refresh_words
        d.shared = _p(self.shared)
        d.epochs, d.loss_every = epochs, loss_every
        d.workers = C.cast(self.workers, P)
        d.n_workers = n_workers
        d.loss_by_epoch, d.cells_by_epoch = _p(self.loss), _p(self.cells)
        d.update = int(update)
        d.trace_cap = trace_cap
        d.trace = _p(self.trace) if trace_cap else None
        d.trace_alpha = _p(self.trace_alpha)
        d.trace_count = _p(self.trace_count)
        d.position_mode = int(position_mode)
        d.matmul = MATMUL[matmul] if d.dtype == 0 else 0
        self.d = d

    @property
    def done(self) -> bool:
        return all(w.done for w in self.workers)

    def advance(self, word_budget: int, n_threads: int = 1) -> int:
        before = sum(w.words_read for w in self.workers)
        self.d.word_budget = word_budget
        _lib.or_drive(C.byref(self.d), n_threads)
        return sum(w.words_read for w in self.workers) - before

    def run_to_completion(self, n_threads: int = 1) -> None:
        while not self.done:
            self.advance(2**62, n_threads)

    def stats(self):
        words_trained = sum(w.words_trained for w in self.workers)
        words_read = sum(w.words_read for w in self.workers)
        ls, cs = self.loss.sum(axis=0), self.cells.sum(axis=0)
        loss = [float(a / b) if b else 0.0 for a, b in zip(ls, cs)]
        return words_trained, words_read, loss

    def worker_trace(self, w: int):
        n = min(int(self.trace_count[w]), self.trace_cap)
        return self.trace[w, :n], self.trace_alpha[w, :n]
