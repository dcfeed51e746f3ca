"""Device RNG cost alone and its interaction with the adaptive loop.
   python tools/rng_probe.py"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2310_09417_b200 as rs  # noqa: E402
from paper_2310_09417_b200 import _device  # noqa: E402

s = rs.RngStream(0).child(3)
for n, ell in [(20000, 64), (4096, 256), (16384, 1024), (65536, 64)]:
    out = torch.empty((n, ell), dtype=torch.float64, device="cuda")
    _device.gaussian(s, n, ell, out=out)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        _device.gaussian(s, n, ell, out=out, status=torch.zeros(1, dtype=torch.int32, device="cuda"))
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    print(f"gaussian {n}x{ell}: {ms:.3f} ms  ({n * ell / ms / 1e6:.1f} Gnormal/s)", flush=True)
