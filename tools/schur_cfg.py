"""Schur GEMM time for the library's row-major DMMA config and the experiment builds.
   python tools/schur_cfg.py [lib.so ...]"""
import os
import sys

import torch

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
from paper_2310_09417_b200 import _device, _lib  # noqa: E402

libs = sys.argv[1:] or [None]
m, b = 20000, 64
for path in libs:
    if path:
        _lib._lib = None
        _lib.load(path)
    ws, st = _device.workspace().data_ptr(), _device.stream_handle()
    Y = torch.randn(m, b, dtype=torch.float64, device="cuda")
    perm = torch.randperm(m, device="cuda")
    S = torch.empty(m, b, dtype=torch.float64, device="cuda")
    row = []
    for k in (2000, 5000, 8000, 11000, 14000):
        R = m - k
        T = torch.randn(R, k, dtype=torch.float64, device="cuda")
        f = lambda: _lib.call("rs_schur_block", m, k, b, Y.data_ptr(), b, perm.data_ptr(), T.data_ptr(), k,  # noqa: E731
                              S.data_ptr(), b, None, ws, st)
        f()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10):
            f()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 10
        row.append(f"k={k}:{ms:.3f}ms/{2 * R * k * b / ms / 1e9:.1f}TF")
        del T
    print(path or "librskel.so", " ".join(row), flush=True)
