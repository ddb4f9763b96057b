"""Diagnostic: does the configs[1] update kernel's time depend on where the models land in
HBM?  Runs one microbench shape repeatedly in one process: fresh, after a dummy allocation
shifts the allocator, and after empty_cache.  Prints us/launch per trial."""
import sys
import os
import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1604_04661_b200.kernel_batched import DeviceWindowBatch, WindowBatch, update_windows
from paper_1604_04661_b200.model import DeviceModel, EmbeddingModel


def trial(base_in, base_out, dwb, steps=30):
    src = DeviceModel.from_host(EmbeddingModel(base_in, base_out))
    dst = src.clone()
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
    for _ in range(3):
        update_windows(dst, dwb, 0.025, src=src)
    ts = []
    for _ in range(steps):
        flush.add_(1.0)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        update_windows(dst, dwb, 0.025, src=src)
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b) * 1e3)
    addr = (src.m_in.data_ptr(), src.m_out.data_ptr(), dst.m_in.data_ptr(), dst.m_out.data_ptr())
    return float(np.median(ts)), [hex(x) for x in addr]


def main(d=300, w=5, k=10, n_win=65536, V=100_000):
    rng = np.random.default_rng(1)
    ranks = np.arange(1, V + 1, dtype=np.float64)
    pz = 1.0 / ranks
    pz /= pz.sum()
    pn = pz ** 0.75
    pn /= pn.sum()
    sig = d ** -0.25
    base_in = (rng.normal(size=(V, d)) * sig).astype(np.float32)
    base_out = (rng.normal(size=(V, d)) * sig).astype(np.float32)
    off = np.arange(0, 2 * w * (n_win + 1), 2 * w, dtype=np.int32)
    ins = rng.choice(V, size=int(off[-1]), p=pz).astype(np.int32)
    tgt = rng.choice(V, size=n_win, p=pz).astype(np.int32)
    negs = rng.choice(V, size=(n_win, k), p=pn).astype(np.int32)
    bad = negs == tgt[:, None]
    while bad.any():
        negs[bad] = rng.choice(V, size=int(bad.sum()), p=pn)
        bad = negs == tgt[:, None]
    outs = np.concatenate([tgt[:, None], negs], axis=1).astype(np.int32)
    dwb = DeviceWindowBatch(WindowBatch(off, ins, outs))
    print("fresh", *trial(base_in, base_out, dwb), flush=True)
    print("again", *trial(base_in, base_out, dwb), flush=True)
    keep = [torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device="cuda") for _ in range(3)]
    print("after 768MB held", *trial(base_in, base_out, dwb), flush=True)
    del keep
    torch.cuda.empty_cache()
    print("after empty_cache", *trial(base_in, base_out, dwb), flush=True)
    keep = [torch.empty(100 * 1024 * 1024 + 4096 * i, dtype=torch.uint8, device="cuda") for i in range(5)]
    print("after odd allocations", *trial(base_in, base_out, dwb), flush=True)


if __name__ == "__main__":
    main(*[int(x) for x in sys.argv[1:]])
