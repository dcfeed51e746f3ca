"""Can the panel (latency-bound, cooperative) and the next block's Schur GEMM (DMMA-bound)
share the GPU?  Times each alone and both on two streams (panel launched first), at cfg2-like
sizes.  python tools/overlap_probe.py"""
import os
import sys

import torch

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
from paper_2310_09417_b200 import _device, _lib  # noqa: E402

m, b = 20000, 64
dev = torch.device("cuda")
for k in (4000, 8000, 12000):
    R = m - k
    S0 = torch.randn(R, b, dtype=torch.float64, device=dev)
    Ss = [S0.clone() for _ in range(10)]
    perm_out = torch.empty(R, dtype=torch.int64, device=dev)
    nc = torch.zeros(1, dtype=torch.int32, device=dev)
    Y = torch.randn(m, b, dtype=torch.float64, device=dev)
    perm = torch.randperm(m, device=dev)
    T = torch.randn(R, k, dtype=torch.float64, device=dev)
    X = torch.empty(m, b, dtype=torch.float64, device=dev)
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    ws1, ws2 = _device.workspace(1).data_ptr(), _device.workspace(2).data_ptr()

    def panel(i, st):
        _lib.call("rs_panel_lupp", Ss[i].data_ptr(), b, R, b, perm_out.data_ptr(), nc.data_ptr(), ws1, st.cuda_stream)

    def schur(st):
        _lib.call("rs_schur_block", m, k, b, Y.data_ptr(), b, perm.data_ptr(), T.data_ptr(), k, X.data_ptr(), b,
                  None, ws2, st.cuda_stream)

    def timed(fn):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / 10

    def only_panel():
        for i in range(10):
            panel(i, torch.cuda.current_stream())

    def only_schur():
        for i in range(10):
            schur(torch.cuda.current_stream())

    def both():
        cur = torch.cuda.current_stream()
        for i in range(10):
            s1.wait_stream(cur)
            s2.wait_stream(cur)
            panel(i, s1)
            schur(s2)
            cur.wait_stream(s1)
            cur.wait_stream(s2)

    for f in (only_panel, only_schur, both):
        f()
    tp, ts, tb = timed(only_panel), timed(only_schur), timed(both)
    print(f"k={k} R={R}: panel {1e3 * tp:.0f} us, schur {1e3 * ts:.0f} us, sum {1e3 * (tp + ts):.0f} us, "
          f"both on two streams {1e3 * tb:.0f} us", flush=True)
