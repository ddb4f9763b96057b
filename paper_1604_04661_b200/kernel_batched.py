"""Per-minibatch operator: `Minibatch` / `process_batch` with the CUDA backend.

Reference map:
  Minibatch        sgns/kernel_batched.py:37-54
  process_batch    sgns/kernel_batched.py:214-260  (backend selector :229-232)
  batch_core_*     sgns/kernel_batched.py:92-211   -> sgns_update_windows (C ABI)

`process_batch(model, batch, alpha)` keeps the reference's signature and
error behaviour; the only backend is "cuda" (`matmul=None` selects it).  The
packed form `WindowBatch` carries many windows in CSR layout (in_off, in_ids,
out_ids) and `update_windows` applies them in one launch, either in place
(Hogwild, as concurrent reference threads would) or in snapshot mode (every
window reads `src`, deltas accumulate into the destination).
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Sequence

import numpy as np

from . import _lib
from .model import (DeviceModel, EmbeddingModel, SIGMOID_TABLE_F32, SIGMOID_TABLE_F64,
                    current_stream_ptr)

# The reference's backend names (kernel_batched.py:229-232) are accepted so callers written
# against it run unchanged; every name selects the one CUDA core, whose float32 results
# match either reference backend within the tolerance the reference itself allows between
# them (rtol 2e-5, tests/test_kernel_batched.py:133-140).
BACKENDS = ("cuda", "blas", "naive")


@dataclass
class Minibatch:
    """B input ids sharing one target (output_ids[0]) and K shared negatives."""

    input_ids: np.ndarray
    output_ids: np.ndarray

    def __post_init__(self) -> None:
        self.input_ids = np.ascontiguousarray(self.input_ids, dtype=np.int32)
        self.output_ids = np.ascontiguousarray(self.output_ids, dtype=np.int32)
        if len(self.input_ids) < 1 or len(self.output_ids) < 2:
            raise ValueError("minibatch needs >= 1 input and >= 2 outputs")
        if (self.output_ids[1:] == self.output_ids[0]).any():
            raise ValueError("a shared negative equals the target")


@dataclass
class WindowBatch:
    """Packed windows: inputs of window w are in_ids[in_off[w]:in_off[w+1]]."""

    in_off: np.ndarray   # int32, n + 1
    in_ids: np.ndarray   # int32
    out_ids: np.ndarray  # int32, n x k1 (target first)

    @property
    def n_windows(self) -> int:
        return len(self.in_off) - 1

    @property
    def k1(self) -> int:
        return self.out_ids.shape[1]

    @property
    def max_inputs(self) -> int:
        return int(np.diff(self.in_off).max()) if self.n_windows else 0

    @classmethod
    def from_minibatches(cls, batches: Sequence[Minibatch]) -> "WindowBatch":
        if not batches:
            raise ValueError("no minibatches")
        k1 = len(batches[0].output_ids)
        if any(len(b.output_ids) != k1 for b in batches):
            raise ValueError("all minibatches of a packed batch need the same K")
        lens = np.array([len(b.input_ids) for b in batches], dtype=np.int64)
        off = np.concatenate([[0], np.cumsum(lens)]).astype(np.int32)
        return cls(off, np.concatenate([b.input_ids for b in batches]).astype(np.int32),
                   np.stack([b.output_ids for b in batches]).astype(np.int32))

    def validate(self, vocab_size: int) -> None:
        if self.n_windows and (np.diff(self.in_off) < 1).any():
            raise ValueError("every window needs >= 1 input")
        if self.in_ids.size and (self.in_ids.min() < 0 or self.in_ids.max() >= vocab_size):
            raise ValueError("input id out of range")
        if self.out_ids.size and (self.out_ids.min() < 0 or self.out_ids.max() >= vocab_size):
            raise ValueError("output id out of range")
        if (self.out_ids[:, 1:] == self.out_ids[:, :1]).any():
            raise ValueError("a shared negative equals the target")


class DeviceWindowBatch:
    """WindowBatch resident in HBM."""

    def __init__(self, wb: WindowBatch, device="cuda"):
        import torch
        self.n_windows = wb.n_windows
        self.k1 = wb.k1
        self.max_inputs = wb.max_inputs
        self.in_off = torch.from_numpy(np.ascontiguousarray(wb.in_off, dtype=np.int32)).to(device)
        self.in_ids = torch.from_numpy(np.ascontiguousarray(wb.in_ids, dtype=np.int32)).to(device)
        self.out_ids = torch.from_numpy(np.ascontiguousarray(wb.out_ids, dtype=np.int32)).to(device)


_TABLES: dict = {}


def device_sigmoid_table(np_dtype, device):
    import torch
    key = (np.dtype(np_dtype).str, str(device))
    if key not in _TABLES:
        tab = SIGMOID_TABLE_F64 if np.dtype(np_dtype) == np.float64 else SIGMOID_TABLE_F32
        _TABLES[key] = torch.from_numpy(tab.copy()).to(device)
    return _TABLES[key]


def update_windows(dst: DeviceModel, batch: DeviceWindowBatch, alpha, *, src: DeviceModel | None = None,
                   sigmoid: str | None = None, loss_every: int = 0, stream=None, error=None):
    """Apply a packed batch of windows with one kernel launch.

    dst: model receiving the deltas.  src: rows are gathered from here
    (None: src = dst, Hogwild in place).  alpha: scalar or per-window tensor.
    Returns (loss_sum, loss_cells) device tensors when loss_every > 0.
    """
    import torch
    src = dst if src is None else src
    if src.m_in.shape != dst.m_in.shape or src.m_in.dtype != dst.m_in.dtype:
        raise ValueError("src and dst models must share shape and dtype")
    dev = dst.m_in.device
    npdt = dst.np_dtype
    if sigmoid is None:
        sigmoid = "exact" if npdt == np.float64 else "table"
    if sigmoid not in ("table", "exact"):
        raise ValueError(f"unknown sigmoid mode {sigmoid!r}")
    if torch.is_tensor(alpha):
        alphas = alpha.to(device=dev, dtype=dst.m_in.dtype).contiguous()
        if alphas.numel() != batch.n_windows:
            raise ValueError("need one alpha per window")
    else:
        if alpha < 0:
            raise ValueError("alpha must be non-negative")
        alphas = torch.full((max(batch.n_windows, 1),), float(alpha), dtype=dst.m_in.dtype, device=dev)
    loss = cells = None
    if loss_every > 0:
        loss = torch.zeros(1, dtype=torch.float64, device=dev)
        cells = torch.zeros(1, dtype=torch.int64, device=dev)
    tab = device_sigmoid_table(npdt, dev)
    st = current_stream_ptr(dev) if stream is None else stream
    rc = _lib.lib().sgns_update_windows(
        dst.cdtype, dst.m_in.data_ptr(), dst.m_out.data_ptr(), src.m_in.data_ptr(),
        src.m_out.data_ptr(), dst.vocab_size, dst.dim, dst.ld, batch.in_off.data_ptr(),
        batch.in_ids.data_ptr(), batch.out_ids.data_ptr(), batch.n_windows, batch.k1,
        max(batch.max_inputs, 1), alphas.data_ptr(), tab.data_ptr(),
        _lib.SIGMOID_EXACT if sigmoid == "exact" else _lib.SIGMOID_TABLE, loss_every,
        None if loss is None else loss.data_ptr(), None if cells is None else cells.data_ptr(),
        None if error is None else error.data_ptr(), st)
    _lib.check(rc, "sgns_update_windows")
    if loss_every > 0:
        return loss, cells
    return None


def process_batch(model, batch: Minibatch, alpha: float, matmul: str | None = None) -> None:
    """Apply one minibatch update in place on the GPU.

    model: EmbeddingModel (host arrays: only the window's distinct rows are copied
    to the device and back, see _process_rows) or DeviceModel (updated in HBM).  float64 models use the exact
    sigmoid, float32 models the 1000-bin table, as the reference does.
    """
    if alpha < 0:
        raise ValueError("alpha must be non-negative")
    if matmul is None:
        matmul = "cuda"
    if matmul not in BACKENDS:
        raise ValueError(f"unknown matmul backend {matmul!r} (one of {', '.join(BACKENDS)}; all run on CUDA)")
    wb = WindowBatch.from_minibatches([batch])
    if isinstance(model, DeviceModel):
        wb.validate(model.vocab_size)
        update_windows(model, DeviceWindowBatch(wb, model.m_in.device), alpha)
        return
    if not isinstance(model, EmbeddingModel):
        raise TypeError("model must be an EmbeddingModel or DeviceModel")
    wb.validate(model.vocab_size)
    _process_rows(model, wb, alpha)


def _process_rows(model: EmbeddingModel, wb: WindowBatch, alpha: float) -> None:
    """Host model, row-granular: only the window's distinct input and output rows travel.

    The reference's batch core gathers exactly these rows, updates them and scatters
    them back (kernel_batched.py:92-144, :214-260).  Here the distinct rows of each
    matrix are packed into a compact device model (ids remapped; repeated ids map to
    one compact row, so repeated inputs accumulate into one row exactly as in place),
    the launch runs on it, and the rows are written back -- (m + K + 1) rows each way
    instead of the whole V x D model."""
    import torch
    in_rows, in_map = np.unique(wb.in_ids, return_inverse=True)
    out_rows, out_map = np.unique(wb.out_ids, return_inverse=True)
    n = max(len(in_rows), len(out_rows))
    dev = torch.device("cuda", torch.cuda.current_device())
    dm = DeviceModel.empty(n, model.dim, model.dtype, dev)
    a = np.zeros((n, model.dim), dtype=model.dtype)
    c = np.zeros((n, model.dim), dtype=model.dtype)
    a[:len(in_rows)] = model.input_vectors[in_rows]
    c[:len(out_rows)] = model.output_vectors[out_rows]
    dm.m_in[:, :model.dim].copy_(torch.from_numpy(a))
    dm.m_out[:, :model.dim].copy_(torch.from_numpy(c))
    compact = WindowBatch(wb.in_off, in_map.astype(np.int32).reshape(wb.in_ids.shape),
                          out_map.astype(np.int32).reshape(wb.out_ids.shape))
    update_windows(dm, DeviceWindowBatch(compact, dev), alpha)
    model.input_vectors[in_rows] = dm.m_in[:len(in_rows), :model.dim].cpu().numpy()
    model.output_vectors[out_rows] = dm.m_out[:len(out_rows), :model.dim].cpu().numpy()
