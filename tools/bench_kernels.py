"""Microbenchmarks of the individual skeleton kernels (CUDA events, warm).

  PYTHONPATH=. python tools/bench_kernels.py [panel|gemm|all]
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", "oracle"))
from paper_2310_09417_b200 import _device, _lib  # noqa: E402


def timeit(fn, reps=20, warm=3):
    for _ in range(warm):
        fn()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def bench_panel():
    ws = _device.workspace()
    for R in (2000, 6000, 20000, 65472):
        s0 = torch.randn(R, 64, dtype=torch.float64, device="cuda")
        S = s0.clone()
        perm = torch.empty(R, dtype=torch.int64, device="cuda")
        nc = torch.empty(1, dtype=torch.int32, device="cuda")

        def run():
            S.copy_(s0)
            _lib.call("rs_panel_lupp", S.data_ptr(), 64, R, 64, perm.data_ptr(), nc.data_ptr(),
                      ws.data_ptr(), _device.stream_handle())

        ms = timeit(run)
        copy_ms = timeit(lambda: S.copy_(s0))
        import randskel_oracle as orc
        if R <= 20000:
            _, _, p0, _ = orc.lupp(s0.cpu().numpy())
            ok = np.array_equal(perm.cpu().numpy(), p0)
        else:
            ok = "n/a"
        print(f"panel R={R:6d} w=64: {1e3 * (ms - copy_ms):8.1f} us/panel "
              f"({1e3 * (ms - copy_ms) / 64:.2f} us/column) ncols={int(nc.item())} perm==oracle {ok}")


def bench_gemm():
    ws = _device.workspace()
    st = _device.stream_handle()
    n = 20000
    a = torch.randn(n, n, dtype=torch.float64, device="cuda")
    om = torch.randn(n, 64, dtype=torch.float64, device="cuda")
    y = torch.empty(n, 64, dtype=torch.float64, device="cuda")
    for colmajor in (1, 0):
        ms = timeit(lambda: _lib.call("rs_sketch_gemm", n, n, 64, a.data_ptr(), n, colmajor,
                                      om.data_ptr(), 64, y.data_ptr(), 64, ws.data_ptr(), st), reps=10)
        print(f"sketch gemm 20000^2 x 64 colmajor={colmajor}: {ms:.3f} ms "
              f"{2 * n * n * 64 / ms / 1e9:.1f} TF/s")
    ref = a.T @ om
    _lib.call("rs_sketch_gemm", n, n, 64, a.data_ptr(), n, 1, om.data_ptr(), 64, y.data_ptr(), 64,
              ws.data_ptr(), st)
    print("  max rel err vs cuBLAS:", float((y - ref).abs().max() / ref.abs().max()))
    ms = timeit(lambda: a.T @ om, reps=10)
    print(f"cuBLAS a.T@om: {ms:.3f} ms {2 * n * n * 64 / ms / 1e9:.1f} TF/s")
    # Schur-shaped: M = m - k rows, K = k, N = 64, gathered B / Cin rows
    for k in (2000, 7000, 14000):
        R = n - k
        T = torch.randn(R, k, dtype=torch.float64, device="cuda")
        perm = torch.randperm(n, device="cuda")
        S = torch.empty(R, 64, dtype=torch.float64, device="cuda")
        e2 = torch.empty(1, dtype=torch.float64, device="cuda")
        ms = timeit(lambda: _lib.call("rs_schur_block", n, k, 64, y.data_ptr(), 64, perm.data_ptr(),
                                      T.data_ptr(), k, S.data_ptr(), 64, e2.data_ptr(), ws.data_ptr(), st),
                    reps=10)
        print(f"schur k={k:5d}: {ms:.3f} ms {2 * R * k * 64 / ms / 1e9:.1f} TF/s")
        # absorb: T' = T[Q] - W T[P], with W = L_r L1^-1
        Sx = torch.randn(R, 64, dtype=torch.float64, device="cuda") * 0.1
        sub = torch.randperm(R, device="cuda")
        Tn = torch.empty((R - 64) * (k + 64), dtype=torch.float64, device="cuda")
        pn = torch.empty(n, dtype=torch.int64, device="cuda")
        ms = timeit(lambda: _lib.call("rs_absorb_block", n, k, 64, Sx.data_ptr(), 64, sub.data_ptr(),
                                      T.data_ptr(), k, Tn.data_ptr(), perm.data_ptr(), pn.data_ptr(),
                                      ws.data_ptr(), st), reps=10)
        fl = 2 * (R - 64) * 64 * k
        by = 16 * (R - 64) * k
        print(f"absorb k={k:5d}: {ms:.3f} ms {fl / ms / 1e9:.1f} TF/s {by / ms / 1e6:.0f} GB/s")
        What = torch.randn(R - 64, 64, dtype=torch.float64, device="cuda")
        ms = timeit(lambda: _lib.call("rs_rank_update", R - 64, k, 64, What.data_ptr(), 64, T.data_ptr(), k,
                                      sub.data_ptr(), T.data_ptr(), k, sub.data_ptr() + 8 * 64,
                                      Tn.data_ptr(), k, st), reps=10)
        print(f"  rank_update only: {ms:.3f} ms {fl / ms / 1e9:.1f} TF/s {by / ms / 1e6:.0f} GB/s")
        Tref = T[sub[64:]] - What @ T[sub[:64]]
        print("  rank_update max err:", float((Tn[: (R - 64) * k].view(R - 64, k) - Tref).abs().max()))
        # absorb(t) + Schur(t+1): one call (rs_absorb_schur; RSKEL_FUSED=0 -> two passes)
        Sn = torch.empty(R, 64, dtype=torch.float64, device="cuda")
        y2 = torch.randn(n, 64, dtype=torch.float64, device="cuda")
        ms = timeit(lambda: _lib.call("rs_absorb_schur", n, k, 64, Sx.data_ptr(), 64, sub.data_ptr(),
                                      T.data_ptr(), k, Tn.data_ptr(), perm.data_ptr(), pn.data_ptr(),
                                      y2.data_ptr(), 64, Sn.data_ptr(), e2.data_ptr(), ws.data_ptr(), st),
                    reps=10)
        print(f"  absorb+schur k={k:5d}: {ms:.3f} ms {2 * fl / ms / 1e9:.1f} TF/s")
        linv = torch.empty(64, 64, dtype=torch.float64, device="cuda")
        ms = timeit(lambda: _lib.call("rs_trinv", Sx.data_ptr(), 64, 1, sub.data_ptr(), 64, 1, 1,
                                      linv.data_ptr(), 64, st), reps=10)
        print(f"  trinv 64: {1e3 * ms:.1f} us")


if __name__ == "__main__":
    what = sys.argv[1] if len(sys.argv) > 1 else "all"
    if what in ("panel", "all"):
        bench_panel()
    if what in ("gemm", "all"):
        bench_gemm()
