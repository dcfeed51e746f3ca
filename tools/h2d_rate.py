"""Host->device and device->host rates: pinned DMA, the pageable staging ring, and the pageable
readback.  python tools/h2d_rate.py"""
import os
import sys
import time

import numpy as np
import torch

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
from paper_2310_09417_b200 import _device  # noqa: E402

n = 20000
h = np.random.default_rng(0).standard_normal((n, n))
pin = torch.from_numpy(h).pin_memory()
dev = torch.empty((n, n), dtype=torch.float64, device="cuda")
gb = h.nbytes / 1e9
for rep in range(3):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    dev.copy_(pin, non_blocking=True); torch.cuda.synchronize(); t1 = time.perf_counter()
    _device.h2d_rows(h, lambda r0, r1, ev: None, out=dev); torch.cuda.synchronize(); t2 = time.perf_counter()
    out = _device.d2h_pageable(dev); t3 = time.perf_counter()
    pin.copy_(dev, non_blocking=True); torch.cuda.synchronize(); t4 = time.perf_counter()
    print(f"rep {rep}: pinned H2D {gb / (t1 - t0):.1f} GB/s, pageable ring H2D {gb / (t2 - t1):.1f} GB/s, "
          f"pageable D2H {gb / (t3 - t2):.1f} GB/s, pinned D2H {gb / (t4 - t3):.1f} GB/s", flush=True)
    del out

# in-place page-locking of the caller's arrays instead of staging
cudart = torch.cuda.cudart()
for rep in range(3):
    t0 = time.perf_counter()
    rc = cudart.cudaHostRegister(h.ctypes.data, h.nbytes, 0)
    t1 = time.perf_counter()
    hv = torch.from_numpy(h)
    dev.copy_(hv, non_blocking=True); torch.cuda.synchronize(); t2 = time.perf_counter()
    cudart.cudaHostUnregister(h.ctypes.data); t3 = time.perf_counter()
    o = np.empty((n, n)); t4 = time.perf_counter()
    cudart.cudaHostRegister(o.ctypes.data, o.nbytes, 0); t5 = time.perf_counter()
    torch.from_numpy(o).copy_(dev, non_blocking=True); torch.cuda.synchronize(); t6 = time.perf_counter()
    cudart.cudaHostUnregister(o.ctypes.data); t7 = time.perf_counter()
    print(f"rep {rep}: rc {rc} register {1e3*(t1-t0):.1f} ms, H2D {1e3*(t2-t1):.1f} ms, unregister {1e3*(t3-t2):.1f} ms | "
          f"fresh out: register {1e3*(t5-t4):.1f} ms, D2H {1e3*(t6-t5):.1f} ms, unregister {1e3*(t7-t6):.1f} ms", flush=True)
    del o

# host-side copy alone: pageable -> reused pinned 32 MB buffers with the thread pool (no DMA)
from paper_2310_09417_b200 import _omega  # noqa: E402

pool = _omega._pool()
bufs = [torch.empty(32 << 20, dtype=torch.uint8, pin_memory=True).numpy() for _ in range(4)]
src = h.reshape(-1).view(np.uint8)
for nthr in (8, 16):
    t0 = time.perf_counter()
    for i, c0 in enumerate(range(0, src.size, 32 << 20)):
        c1 = min(src.size, c0 + (32 << 20))
        buf = bufs[i % 4]
        part = -(-(c1 - c0) // nthr)
        list(pool.map(lambda q: np.copyto(buf[q:q + part][: max(0, min(part, c1 - c0 - q))], src[c0 + q:c0 + q + part][: max(0, min(part, c1 - c0 - q))]), range(0, c1 - c0, part)))
    t1 = time.perf_counter()
    print(f"host copy pageable->pinned, {nthr} threads: {gb / (t1 - t0):.1f} GB/s", flush=True)
