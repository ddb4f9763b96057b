"""Model parameters: host `EmbeddingModel` (reference API) and its HBM twin `DeviceModel`.

Reference map:
  EmbeddingModel            sgns/model.py:29-53
  init_model                sgns/model.py:64-74   (here: sgns_init_model on device, bit-identical)
  sigmoid / sigmoid table   sgns/model.py:77-115  (host table uploaded; index math stays float64)

HBM layout: each matrix is a (V, ld) row-major tensor with ld = dim rounded up
so a row is a whole number of 32-byte sectors, and for float32 a whole number
of 128-byte lines when that costs at most 12.5% (ld = 320 at d = 300); padding
columns are zero and stay zero.  Dims that are multiples of 64 get the fast
path's whole-slot variant automatically.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from . import _lib

SIGMOID_RANGE = 6.0
SIGMOID_BINS = 1000


@dataclass
class EmbeddingModel:
    input_vectors: np.ndarray  # V x D
    output_vectors: np.ndarray  # V x D

    @property
    def vocab_size(self) -> int:
        return self.input_vectors.shape[0]

    @property
    def dim(self) -> int:
        return self.input_vectors.shape[1]

    @property
    def dtype(self) -> np.dtype:
        return self.input_vectors.dtype

    def copy(self) -> "EmbeddingModel":
        return EmbeddingModel(self.input_vectors.copy(), self.output_vectors.copy())

    def assert_finite(self) -> None:
        if not np.isfinite(self.input_vectors).all():
            raise FloatingPointError("non-finite entries in input_vectors")
        if not np.isfinite(self.output_vectors).all():
            raise FloatingPointError("non-finite entries in output_vectors")


def sigmoid(x):
    """Exact, numerically stable logistic function (scalar or array)."""
    if np.isscalar(x) or np.ndim(x) == 0:
        x = float(x)
        if x >= 0:
            return 1.0 / (1.0 + math.exp(-x))
        ex = math.exp(x)
        return ex / (1.0 + ex)
    x = np.asarray(x, dtype=np.float64)
    out = np.empty_like(x)
    pos = x >= 0
    out[pos] = 1.0 / (1.0 + np.exp(-x[pos]))
    ex = np.exp(x[~pos])
    out[~pos] = ex / (1.0 + ex)
    return out


def build_sigmoid_table(dtype=np.float32) -> np.ndarray:
    """Left-edge sigmoid over [-6, 6) in 1000 bins (host float64, cast once)."""
    edges = -SIGMOID_RANGE + np.arange(SIGMOID_BINS) * (2.0 * SIGMOID_RANGE / SIGMOID_BINS)
    return sigmoid(edges).astype(dtype)


SIGMOID_TABLE_F32 = build_sigmoid_table(np.float32)
SIGMOID_TABLE_F64 = build_sigmoid_table(np.float64)


import os

# Row stride policy: rows are a whole number of 32-byte sectors (a 16-byte cp.async whose
# shared-memory destination and global source sit at different offsets within a sector
# fetches one sector per lane instead of per pair of lanes, tools/probes/ldgsts_probe.cu),
# and for float32 a whole number of 128-byte lines when that costs at most LD_LINE_WASTE of
# the model, so that a warp-wide gather / RED.128 covers whole lines (d = 300 -> ld = 320:
# 4 + 4 + 2 L2 requests per row instead of 5 + 5 + 2..3; +7% words/s on the 1M-word model).
# The production kernel only touches the dim columns that hold data; the pad stays zero.
LD_LINE_WASTE = float(os.environ.get("SGNS_LD_LINE_WASTE", "0.125"))


def padded_ld(dim: int, dtype) -> int:
    """Row stride in elements: whole 32-byte sectors, whole 128-byte lines when cheap."""
    per32 = 32 // np.dtype(dtype).itemsize
    ld = -(-dim // per32) * per32
    if np.dtype(dtype) == np.float32:
        line = -(-dim // 32) * 32
        if (line - dim) / dim <= LD_LINE_WASTE:
            ld = line
    return ld


def _torch():
    import torch
    if not torch.cuda.is_available():
        raise RuntimeError("paper_1604_04661_b200 needs a CUDA device (no CPU fallback)")
    return torch


def _tdtype(torch, dtype):
    return torch.float64 if np.dtype(dtype) == np.float64 else torch.float32


def _cdtype(dtype) -> int:
    return _lib.SGNS_F64 if np.dtype(dtype) == np.float64 else _lib.SGNS_F32


def current_stream_ptr(device=None) -> int:
    torch = _torch()
    return torch.cuda.current_stream(device).cuda_stream


class DeviceModel:
    """M_in / M_out resident in HBM as (V, ld) tensors."""

    def __init__(self, m_in, m_out, dim: int, storage=None):
        self.m_in = m_in
        self.m_out = m_out
        self.dim = dim
        # (2, V, ld) tensor holding both matrices back to back when allocated here: a
        # full-model average is then a single collective on one contiguous buffer
        self.storage = storage

    @property
    def vocab_size(self) -> int:
        return self.m_in.shape[0]

    @property
    def ld(self) -> int:
        return self.m_in.shape[1]

    @property
    def np_dtype(self):
        import torch
        return np.float64 if self.m_in.dtype == torch.float64 else np.float32

    @property
    def cdtype(self) -> int:
        return _cdtype(self.np_dtype)

    @classmethod
    def empty(cls, vocab_size: int, dim: int, dtype=np.float32, device="cuda") -> "DeviceModel":
        torch = _torch()
        ld = padded_ld(dim, dtype)
        td = _tdtype(torch, dtype)
        st = torch.zeros((2, vocab_size, ld), dtype=td, device=device)
        return cls(st[0], st[1], dim, st)

    @classmethod
    def from_host(cls, model: EmbeddingModel, device="cuda") -> "DeviceModel":
        torch = _torch()
        dm = cls.empty(model.vocab_size, model.dim, model.dtype, device)
        dm.m_in[:, :model.dim].copy_(torch.from_numpy(np.ascontiguousarray(model.input_vectors)))
        dm.m_out[:, :model.dim].copy_(torch.from_numpy(np.ascontiguousarray(model.output_vectors)))
        return dm

    def to_host(self) -> EmbeddingModel:
        return EmbeddingModel(self.m_in[:, :self.dim].cpu().numpy().copy(),
                              self.m_out[:, :self.dim].cpu().numpy().copy())

    def copy_to_host(self, model: EmbeddingModel) -> None:
        model.input_vectors[...] = self.m_in[:, :self.dim].cpu().numpy()
        model.output_vectors[...] = self.m_out[:, :self.dim].cpu().numpy()

    def clone(self) -> "DeviceModel":
        if self.storage is not None:
            st = self.storage.clone()
            return DeviceModel(st[0], st[1], self.dim, st)
        return DeviceModel(self.m_in.clone(), self.m_out.clone(), self.dim)


def init_device_model(vocab_size: int, dim: int, seed: int, dtype=np.float32,
                      device="cuda") -> DeviceModel:
    """init_model on device: U(-0.5/D, 0.5/D) from splitmix stream (seed, 0x1017), M_out = 0."""
    if vocab_size < 1 or dim < 1:
        raise ValueError("vocab_size and dim must be positive")
    dm = DeviceModel.empty(vocab_size, dim, dtype, device)
    rc = _lib.lib().sgns_init_model(_cdtype(dtype), dm.m_in.data_ptr(), dm.m_out.data_ptr(),
                                    vocab_size, dim, dm.ld, seed & (2**64 - 1),
                                    current_stream_ptr(dm.m_in.device))
    _lib.check(rc, "sgns_init_model")
    return dm


def init_model(vocab_size: int, dim: int, seed: int, dtype=np.float32) -> EmbeddingModel:
    """Reference-compatible init_model (host arrays), generated on the device."""
    return init_device_model(vocab_size, dim, seed, dtype).to_host()


def sigmoid_table_device(dtype, device="cuda"):
    torch = _torch()
    tab = SIGMOID_TABLE_F64 if np.dtype(dtype) == np.float64 else SIGMOID_TABLE_F32
    return torch.from_numpy(tab.copy()).to(device)


# ------------------------------------------------------------------- vector files ----
class ModelFormatError(ValueError):
    """Vector file does not match the expected layout (model.py:22-23)."""


def save_model(model, vocab, path: str, binary: bool = False) -> None:
    """Write input_vectors as a word2vec text/binary file (model.py:118-139), byte-identical.

    model: EmbeddingModel (host float32/float64) or DeviceModel (float32 rows are
    streamed device -> host by the writer)."""
    import ctypes as C
    if model.vocab_size != vocab.size:
        raise ValueError(f"model has {model.vocab_size} rows but vocabulary has {vocab.size}")
    enc = [t.encode("utf-8") for t in vocab.tokens]
    offs = np.zeros(len(enc) + 1, dtype=np.int64)
    offs[1:] = np.cumsum([len(t) for t in enc])
    blob = C.create_string_buffer(b"".join(enc), max(int(offs[-1]), 1))
    if isinstance(model, DeviceModel):
        rows, ld, on_dev, keep = model.m_in.data_ptr(), model.ld, 1, model.m_in
        dt = model.cdtype
        import torch
        torch.cuda.synchronize(model.m_in.device)
    else:
        f64 = model.input_vectors.dtype == np.float64
        arr = np.ascontiguousarray(model.input_vectors, dtype=np.float64 if f64 else np.float32)
        rows, ld, on_dev, keep = arr.ctypes.data, arr.shape[1], 0, arr
        dt = _lib.SGNS_F64 if f64 else _lib.SGNS_F32
    rc = _lib.lib().sgns_write_vectors(path.encode(), C.addressof(blob), offs.ctypes.data, vocab.size,
                                       model.dim, rows, ld, int(binary), on_dev, dt)
    del keep
    if rc == -5:
        raise OSError(f"cannot write {path}")
    _lib.check(rc, "sgns_write_vectors")


def _header(path: str) -> tuple[int, int, int]:
    """(V, D, header length in bytes): the native parser, else Python's int()/split() rules
    for the first line (sgns/model.py:140-150 semantics)."""
    import ctypes as C
    v, d, n = C.c_int64(0), C.c_int32(0), C.c_int64(0)
    rc = _lib.lib().sgns_vectors_header(path.encode(), C.byref(v), C.byref(d), C.byref(n))
    if rc == -5:
        raise FileNotFoundError(path)
    if rc == 0:
        return v.value, d.value, n.value
    with open(path, "rb") as fh:
        first = fh.readline()
    bad = ModelFormatError(f"{path}: malformed header {first!r}")
    try:
        words = first.decode("utf-8").split()
        dims = [int(x) for x in words] if len(words) == 2 else None
    except (UnicodeDecodeError, ValueError):
        dims = None
    if not dims or min(dims) < 1:
        raise bad from None
    return dims[0], dims[1], len(first)


def detect_format(path: str) -> bool:
    """True when the payload looks binary: the first row, decoded and whitespace-split,
    must hold a token and D numbers to count as text (sgns/model.py:153-172 rule)."""
    import ctypes as C
    _, d, hdr = _header(path)
    out = C.c_int32(0)
    rc = _lib.lib().sgns_vectors_sniff(path.encode(), hdr, d, C.byref(out))
    if rc == 0:
        return bool(out.value)
    _lib.check(rc if rc < 0 else 0, "sgns_vectors_sniff")
    with open(path, "rb") as fh:  # a probe field only Python's float() can judge
        fh.seek(hdr)
        fields = fh.read(16 * d + 64).decode("utf-8").split()
    for f in fields[1:d + 1]:
        try:
            float(f)
        except ValueError:
            return True
    return False


def _python_row(path: str, binary: bool, offset: int, d: int, row: int, vocab: int):
    """One row the native parser handed back, under Python's rules: (token, values, next
    offset) or the exception the reference raises for it."""
    with open(path, "rb") as fh:
        fh.seek(offset)
        if binary:  # only an undecodable token comes back here
            raw = fh.read()
            return raw[:raw.index(b" ")].decode("utf-8"), None, None
        raw = fh.read()
    # Python text mode: universal newlines, the row ends at \n, \r\n or \r
    cut = len(raw)
    for sep in (b"\n", b"\r"):
        k = raw.find(sep)
        if 0 <= k < cut:
            cut = k
    nxt = offset + cut + (2 if raw[cut:cut + 2] == b"\r\n" else 1 if cut < len(raw) else 0)
    line = raw[:cut].decode("utf-8")
    cols = line.split(" ")
    if len(cols) - 1 != d:
        raise ModelFormatError(f"{path}: dimension mismatch at word {row}: expected {d} values, got {len(cols) - 1}")
    return cols[0], np.array([float(x) for x in cols[1:]], dtype=np.float32), nxt


def load_model(path: str, binary: bool | None = None):
    """Read a vector file back (sgns/model.py:175-225): rows parsed natively
    (sgns_parse_vectors), output_vectors come back zero, counts are ones."""
    import ctypes as C
    from .corpus import Vocabulary
    v, d, hdr = _header(path)
    if binary is None:
        binary = detect_format(path)
    vectors = np.empty((v, d), dtype=np.float32)
    t0 = np.zeros(v, dtype=np.int64)
    t1 = np.zeros(v, dtype=np.int64)
    names: dict[int, str] = {}  # rows that came back through _python_row
    row, off = C.c_int64(0), C.c_int64(hdr)
    L = _lib.lib()
    while True:
        rc = L.sgns_parse_vectors(path.encode(), int(binary), v, d, vectors.ctypes.data, t0.ctypes.data,
                                  t1.ctypes.data, C.byref(row), C.byref(off))
        if rc == 0:
            break
        if rc == -7:
            raise ModelFormatError(f"{path}: truncated file at word {row.value} of {v}")
        _lib.check(rc if rc < 0 else 0, "sgns_parse_vectors")
        tok, vals, nxt = _python_row(path, binary, off.value, d, row.value, v)
        names[row.value] = tok
        vectors[row.value] = vals
        row.value += 1
        off.value = nxt
    import mmap
    with open(path, "rb") as fh, mmap.mmap(fh.fileno(), 0, access=mmap.ACCESS_READ) as blob:
        tokens = [names[i] if i in names else blob[a:b].decode("utf-8")
                  for i, (a, b) in enumerate(zip(t0.tolist(), t1.tolist()))]
    if binary:
        tokens = [t.lstrip("\n") for t in tokens]
    vocab = Vocabulary(tokens, np.ones(v, dtype=np.int64), {t: i for i, t in enumerate(tokens)}, v)
    return EmbeddingModel(vectors, np.zeros_like(vectors)), vocab


def save_debug(model, vocab, path: str) -> None:
    """Both matrices losslessly (model.py:228-236)."""
    host = model.to_host() if isinstance(model, DeviceModel) else model
    np.savez(path, input_vectors=host.input_vectors, output_vectors=host.output_vectors,
             tokens=np.array(vocab.tokens, dtype=object), counts=vocab.counts)


def load_debug(path: str):
    from .corpus import Vocabulary
    data = np.load(path, allow_pickle=True)
    tokens = list(data["tokens"])
    counts = data["counts"]
    vocab = Vocabulary(tokens, counts, {t: i for i, t in enumerate(tokens)}, int(counts.sum()))
    return EmbeddingModel(data["input_vectors"], data["output_vectors"]), vocab
