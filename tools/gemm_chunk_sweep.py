"""Schur-block GEMM (S = Y[rest] - T Y[top]) time vs the K-chunk length kc, and the sketch GEMM.
   python tools/gemm_chunk_sweep.py"""
import os
import sys

import torch

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
from paper_2310_09417_b200 import _device, _lib  # noqa: E402

m, b = 20000, 64
L = _lib.load()
ws, st = _device.workspace().data_ptr(), _device.stream_handle()
Y = torch.randn(m, b, dtype=torch.float64, device="cuda")
perm = torch.randperm(m, device="cuda")
S = torch.empty(m, b, dtype=torch.float64, device="cuda")


def timeit(f, reps=10):
    f()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        f()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


for k in (512, 2000, 5000, 8000, 11000, 14000):
    R = m - k
    T = torch.randn(R, k, dtype=torch.float64, device="cuda")
    row = []
    for kc in (256, 512, 1024, 2048, 4096, 1 << 20):
        kcc = kc if kc < k else 0
        if kc >= k and kc != (1 << 20):
            continue
        f = lambda: _lib.call("rs_dgemm_ex", R, b, k, kc if kc < (1 << 20) else k, 0, -1.0, T.data_ptr(), k, 0, None,  # noqa: E731
                              Y.data_ptr(), b, perm.data_ptr(), 1.0, Y.data_ptr(), b, perm[k:].data_ptr(), S.data_ptr(),
                              b, ws, st)
        ms = timeit(f)
        row.append(f"kc={'K' if kc == 1 << 20 else kc}:{ms:.3f}ms/{2 * R * k * b / ms / 1e9:.1f}TF")
    dflt = L.rs_gemm_chunk(k)
    cub = timeit(lambda: torch.mm(T, Y[:k]))
    print(f"k={k} R={R} default kc={dflt}: " + " ".join(row) + f"  cuBLAS {cub:.3f}ms/{2 * R * k * b / cub / 1e9:.1f}TF",
          flush=True)
    del T
