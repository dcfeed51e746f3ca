"""Break down the cfg1 end-to-end column_id time (numpy in/out).
   PYTHONPATH=. python tools/e2e_cfg1.py"""
import time

import numpy as np
import torch

import paper_2310_09417_b200 as rs
from paper_2310_09417_b200 import _device

n, k = 4096, 256
a = np.random.default_rng(0).standard_normal((n, n))
spec = rs.SketchSpec("gaussian", n, k)
for rep in range(4):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    A = _device.as_matrix(a)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    r = rs.column_id(A, k, spec, rs.RngStream(0))
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    x = _device.to_output(r.x, "numpy") if isinstance(r.x, torch.Tensor) else r.x
    t3 = time.perf_counter()
    r2 = rs.column_id(a, k, spec, rs.RngStream(0))
    t4 = time.perf_counter()
    print(f"rep {rep}: h2d {1e3 * (t1 - t0):.2f} ms, column_id(device A) {1e3 * (t2 - t1):.2f} ms, "
          f"d2h {1e3 * (t3 - t2):.2f} ms, full numpy call {1e3 * (t4 - t3):.2f} ms")
