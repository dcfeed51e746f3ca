"""Ozaki tcgen05 sketch GEMM: accuracy vs an extended-precision reference, determinism, timing.
  python tools/oz_check.py"""
import os
import sys
import time

import numpy as np
import torch

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
from paper_2310_09417_b200 import _device, _lib  # noqa: E402

L = _lib.load()


def slice_op(X, colmajor, rows, K, S, tile_rows, fp32=False, kc=None):
    kc = kc or L.rs_oz_chunk(K)
    nch = -(-K // kc)
    dig = torch.zeros(L.rs_oz_digits_bytes(rows, K, S, tile_rows), dtype=torch.int8, device="cuda")
    expo = torch.zeros(rows * nch, dtype=torch.int32, device="cuda")
    ld = X.stride(0)  # row stride of the storage (a[i, k] at k*ld + i when colmajor)
    _lib.call("rs_oz_slice", X.data_ptr(), int(fp32), ld, int(colmajor), rows, K, 0, K, kc, S, tile_rows,
              dig.data_ptr(), expo.data_ptr(), None, _device.workspace().data_ptr(), _device.stream_handle())
    return dig, expo, kc


def oz(A, colmajor, om, SA=8, SB=8, fp32=False):
    M, K = A.shape if not colmajor else (A.shape[1], A.shape[0])
    N = om.shape[1]
    ad, ae, kc = slice_op(A, colmajor, M, K, SA, 128, fp32)
    bd, be, _ = slice_op(om, True, N, K, SB, 64)
    Y = torch.empty(M, N, dtype=torch.float64, device="cuda")
    _lib.call("rs_oz_gemm", M, N, K, kc, 0, 1.0, ad.data_ptr(), ae.data_ptr(), SA, bd.data_ptr(), be.data_ptr(), SB,
              0.0, None, 0, Y.data_ptr(), N, _device.workspace().data_ptr(), _device.stream_handle())
    return Y, (ad, ae, bd, be, kc)


def main():
    torch.manual_seed(0)
    for (M, K, N, colmajor, SA, SB) in [(300, 1000, 64, False, 8, 8), (300, 1000, 64, True, 8, 8),
                                        (1000, 5000, 128, True, 8, 8), (2000, 20000, 64, True, 8, 8),
                                        (2000, 20000, 64, True, 7, 7), (2000, 20000, 64, True, 7, 8),
                                        (2000, 65536, 64, True, 8, 8), (2000, 65536, 64, True, 7, 7)]:
        A = torch.randn(M, K, dtype=torch.float64, device="cuda")
        if colmajor:
            A = A.t().contiguous()  # K x M storage: a[i, k] at k*M + i
        om = torch.randn(K, N, dtype=torch.float64, device="cuda") / 8
        Y, _ = oz(A, colmajor, om, SA=SA, SB=SB)
        torch.cuda.synchronize()
        a = (A.t() if colmajor else A).cpu().numpy()
        o = om.cpu().numpy()
        rows = np.arange(0, M, max(1, M // 40))
        ref = np.array([[np.sum(np.longdouble(a[i]) * np.longdouble(o[:, j])) for j in range(N)] for i in rows])
        yd = a[rows] @ o
        y = Y.cpu().numpy()[rows]
        scale = np.abs(a[rows]) @ np.abs(o)
        e_oz = np.max(np.abs(np.longdouble(y) - ref) / scale)
        e_dg = np.max(np.abs(np.longdouble(yd) - ref) / scale)
        print(f"M={M} K={K} N={N} colmajor={colmajor} SA={SA} SB={SB}: max |err|/(|A||O|): ozaki {float(e_oz):.3e}  "
              f"openblas {float(e_dg):.3e}", flush=True)
    # timing at the cfg2 sketch shape
    n = 20000
    A = torch.randn(n, n, dtype=torch.float64, device="cuda")
    om = torch.randn(n, 64, dtype=torch.float64, device="cuda")
    Y, (ad, ae, bd, be, kc) = oz(A, True, om)
    for SA, SB in ((8, 8), (7, 7), (7, 8)):
        for rep in range(2):
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(10):
                _lib.call("rs_oz_gemm", n, 64, n, kc, 0, 1.0, ad.data_ptr(), ae.data_ptr(), SA, bd.data_ptr(),
                          be.data_ptr(), SB, 0.0, None, 0, Y.data_ptr(), 64, _device.workspace().data_ptr(),
                          _device.stream_handle())
            e1.record()
            torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 10
        print(f"oz_gemm 20000x20000x64 SA={SA} SB={SB}: {ms:.3f} ms, {2 * n * n * 64 / ms / 1e9:.1f} fp64-equiv TF/s, "
              f"A-plane bytes {SA * n * n / ms / 1e6:.0f} GB/s", flush=True)
    t0 = time.time()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    slice_op(A, True, n, n, 8, 128)
    e1.record()
    torch.cuda.synchronize()
    print(f"slice 20000^2 fp64 -> 8 planes: {e0.elapsed_time(e1):.2f} ms")


if __name__ == "__main__":
    main()
