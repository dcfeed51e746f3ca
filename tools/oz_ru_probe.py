"""Rank update T' = T[Q] - W_hat T[P] (K = 64) on the int8 tensor cores (Ozaki planes, K padded
to one 128-byte k-block) against the DMMA rank-update kernel, at cfg2 block shapes.
   python tools/oz_ru_probe.py"""
import os
import sys

import torch

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
sys.path.insert(0, os.path.join(REPO, "tools"))
from oz_check import slice_op  # noqa: E402
from paper_2310_09417_b200 import _device, _lib  # noqa: E402

ws, st = _device.workspace().data_ptr(), _device.stream_handle()
dev = torch.device("cuda")
b = 64
for m, k in ((20000, 4000), (20000, 8000), (20000, 12000)):
    R = m - k
    M = R - b
    T = torch.randn(R, k, dtype=torch.float64, device=dev)
    Wh = torch.randn(M, b, dtype=torch.float64, device=dev)
    P = torch.randperm(R, device=dev)[:b]
    Q = torch.randperm(R, device=dev)[:M]
    out = torch.empty(M, k + b, dtype=torch.float64, device=dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)

    def dmma():
        _lib.call("rs_rank_update", M, k, b, Wh.data_ptr(), b, T.data_ptr(), k, P.data_ptr(), T.data_ptr(), k,
                  Q.data_ptr(), out.data_ptr(), k + b, st)

    TP = T[P].contiguous()
    TQ = T[Q].contiguous()

    def ozaki():
        ad, ae, _ = slice_op(Wh, False, M, b, 8, 128, kc=128)
        bd, be, _ = slice_op(TP, True, k, b, 8, 64, kc=128)
        _lib.call("rs_oz_gemm", M, k, b, 128, 0, -1.0, ad.data_ptr(), ae.data_ptr(), 8, bd.data_ptr(), be.data_ptr(),
                  8, 1.0, TQ.data_ptr(), k, out.data_ptr(), k + b, ws, st)

    def gemm_only(ad, ae, bd, be):
        _lib.call("rs_oz_gemm", M, k, b, 128, 0, -1.0, ad.data_ptr(), ae.data_ptr(), 8, bd.data_ptr(), be.data_ptr(),
                  8, 1.0, TQ.data_ptr(), k, out.data_ptr(), k + b, ws, st)

    res = {}
    for name, fn in (("dmma rank update", dmma), ("ozaki slice+gemm", ozaki)):
        fn()
        torch.cuda.synchronize()
        e0.record()
        for _ in range(10):
            fn()
        e1.record()
        torch.cuda.synchronize()
        res[name] = e0.elapsed_time(e1) / 10
    ad, ae, _ = slice_op(Wh, False, M, b, 8, 128, kc=128)
    bd, be, _ = slice_op(TP, True, k, b, 8, 64, kc=128)
    gemm_only(ad, ae, bd, be)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(10):
        gemm_only(ad, ae, bd, be)
    e1.record()
    torch.cuda.synchronize()
    res["ozaki gemm alone"] = e0.elapsed_time(e1) / 10
    ref = TQ - Wh @ TP
    err = (out[:, :k] - ref).abs().max().item() / ref.abs().max().item()
    print(f"m={m} k={k} (M={M}): " + ", ".join(f"{n} {v * 1e3:.0f} us" for n, v in res.items()) + f"; max rel err {err:.1e}",
          flush=True)
