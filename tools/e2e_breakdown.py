"""Where the cfg2 end-to-end time goes: pageable H2D + digit planes, the device loop, the W
readback into a fresh numpy array.  python tools/e2e_breakdown.py"""
import os
import sys
import time

import numpy as np
import torch

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
import paper_2310_09417_b200 as rs  # noqa: E402
from bench import gen_fast_decay_device  # noqa: E402
from paper_2310_09417_b200 import _device, skeleton  # noqa: E402

n = 20000
a = gen_fast_decay_device(n, 1e-16, 0, torch.device("cuda", 0))
h = np.empty((n, n))
h[...] = a.cpu().numpy()
spec = rs.SketchSpec("gaussian", n, 64)
for rep in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    A, planes = skeleton._streamed_planes(h.T)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    res = skeleton._adaptive_device(A, 64, 1e-8, spec, rs.RngStream(0), planes=planes)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    w = res.w if isinstance(res.w, torch.Tensor) else None
    wd = torch.empty((n, res.rank), dtype=torch.float64, device="cuda")
    t3 = time.perf_counter()
    out = _device.d2h_pageable(wd)
    t4 = time.perf_counter()
    print(f"rep {rep}: h2d+planes {1e3 * (t1 - t0):.1f} ms ({3.2 / (t1 - t0):.1f} GB/s), loop {1e3 * (t2 - t1):.1f} ms, "
          f"d2h {1e3 * (t4 - t3):.1f} ms ({wd.numel() * 8 / 1e9 / (t4 - t3):.1f} GB/s), cores {os.cpu_count()}",
          flush=True)
    del out, res, A, planes
