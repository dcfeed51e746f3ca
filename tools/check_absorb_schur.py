"""rs_absorb_schur (one pass over T) against the two-pass kernels on random
data: T' bitwise (same rank-update arithmetic is not required -> allclose),
S' and e2 to rounding.   PYTHONPATH=. python tools/check_absorb_schur.py"""
import os
import subprocess
import sys

import torch

from paper_2310_09417_b200 import _device, _lib

ws = _device.workspace()
st = _device.stream_handle()
torch.manual_seed(0)
for (n, k) in [(3000, 640), (5000, 1998), (20000, 7040)]:
    R = n - k
    y = torch.randn(n, 64, dtype=torch.float64, device="cuda")
    T = torch.randn(R, k, dtype=torch.float64, device="cuda") * 0.3
    perm = torch.randperm(n, device="cuda")
    S = torch.randn(R, 64, dtype=torch.float64, device="cuda") * 0.2
    sub = torch.randperm(R, device="cuda")
    outs = []
    for mode in ("fused", "plain"):
        Tn = torch.zeros((R - 64) * (k + 64), dtype=torch.float64, device="cuda")
        pn = torch.empty(n, dtype=torch.int64, device="cuda")
        Sn = torch.zeros(R, 64, dtype=torch.float64, device="cuda")
        e2 = torch.empty(1, dtype=torch.float64, device="cuda")
        if mode == "fused":
            _lib.call("rs_absorb_schur", n, k, 64, S.data_ptr(), 64, sub.data_ptr(), T.data_ptr(), k,
                      Tn.data_ptr(), perm.data_ptr(), pn.data_ptr(), y.data_ptr(), 64, Sn.data_ptr(),
                      e2.data_ptr(), ws.data_ptr(), st)
        else:
            _lib.call("rs_absorb_block", n, k, 64, S.data_ptr(), 64, sub.data_ptr(), T.data_ptr(), k,
                      Tn.data_ptr(), perm.data_ptr(), pn.data_ptr(), ws.data_ptr(), st)
            _lib.call("rs_schur_block", n, k + 64, 64, y.data_ptr(), 64, pn.data_ptr(), Tn.data_ptr(), k + 64,
                      Sn.data_ptr(), 64, e2.data_ptr(), ws.data_ptr(), st)
        torch.cuda.synchronize()
        outs.append((Tn.clone(), Sn[: R - 64].clone(), float(e2.item()), pn.clone()))
    (T1, S1, e1, p1), (T2, S2, e2_, p2) = outs
    print(f"n={n} k={k}: perm equal {bool(torch.equal(p1, p2))}, T' max diff {float((T1 - T2).abs().max()):.3e}, "
          f"S' max rel diff {float((S1 - S2).abs().max() / S2.abs().max()):.3e}, e2 {e1:.12e} vs {e2_:.12e}")
