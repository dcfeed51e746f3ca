"""Small launch targets for ncu (one kernel family per invocation).

  PYTHONPATH=. python tools/prof_targets.py sketch|schur|rank_update|panel|absorb
"""
import sys

import torch

from paper_2310_09417_b200 import _device, _lib

what = sys.argv[1]
ws = _device.workspace()
st = _device.stream_handle()
n = 20000
k = 7040
R = n - k
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
if what == "sketch":
    a = torch.randn(n, n, dtype=torch.float64, device="cuda")
    om = torch.randn(n, 64, dtype=torch.float64, device="cuda")
    y = torch.empty(n, 64, dtype=torch.float64, device="cuda")
    for _ in range(reps):
        _lib.call("rs_sketch_gemm", n, n, 64, a.data_ptr(), n, 1, om.data_ptr(), 64, y.data_ptr(), 64,
                  ws.data_ptr(), st)
elif what == "fused":
    y = torch.randn(n, 64, dtype=torch.float64, device="cuda")
    T = torch.randn(R, k, dtype=torch.float64, device="cuda")
    perm = torch.randperm(n, device="cuda")
    S = torch.randn(R, 64, dtype=torch.float64, device="cuda") * 0.1
    sub = torch.randperm(R, device="cuda")
    Tn = torch.empty((R - 64) * (k + 64), dtype=torch.float64, device="cuda")
    pn = torch.empty(n, dtype=torch.int64, device="cuda")
    e2 = torch.empty(1, dtype=torch.float64, device="cuda")
    Sn = torch.empty(R, 64, dtype=torch.float64, device="cuda")
    for _ in range(reps):
        _lib.call("rs_absorb_schur", n, k, 64, S.data_ptr(), 64, sub.data_ptr(), T.data_ptr(), k,
                  Tn.data_ptr(), perm.data_ptr(), pn.data_ptr(), y.data_ptr(), 64, Sn.data_ptr(),
                  e2.data_ptr(), ws.data_ptr(), st)
elif what in ("schur", "rank_update", "absorb"):
    y = torch.randn(n, 64, dtype=torch.float64, device="cuda")
    T = torch.randn(R, k, dtype=torch.float64, device="cuda")
    perm = torch.randperm(n, device="cuda")
    S = torch.empty(R, 64, dtype=torch.float64, device="cuda")
    e2 = torch.empty(1, dtype=torch.float64, device="cuda")
    sub = torch.randperm(R, device="cuda")
    Tn = torch.empty((R - 64) * (k + 64), dtype=torch.float64, device="cuda")
    What = torch.randn(R - 64, 64, dtype=torch.float64, device="cuda")
    pn = torch.empty(n, dtype=torch.int64, device="cuda")
    for _ in range(reps):
        if what == "schur":
            _lib.call("rs_schur_block", n, k, 64, y.data_ptr(), 64, perm.data_ptr(), T.data_ptr(), k,
                      S.data_ptr(), 64, e2.data_ptr(), ws.data_ptr(), st)
        elif what == "rank_update":
            _lib.call("rs_rank_update", R - 64, k, 64, What.data_ptr(), 64, T.data_ptr(), k,
                      sub.data_ptr(), T.data_ptr(), k, sub.data_ptr() + 8 * 64, Tn.data_ptr(), k, st)
        else:
            _lib.call("rs_absorb_block", n, k, 64, S.data_ptr(), 64, sub.data_ptr(), T.data_ptr(), k,
                      Tn.data_ptr(), perm.data_ptr(), pn.data_ptr(), ws.data_ptr(), st)
elif what == "panel":
    Rp = int(sys.argv[3]) if len(sys.argv) > 3 else 20000
    s0 = torch.randn(Rp, 64, dtype=torch.float64, device="cuda")
    perm = torch.empty(Rp, dtype=torch.int64, device="cuda")
    nc = torch.empty(1, dtype=torch.int32, device="cuda")
    for _ in range(reps):
        S = s0.clone()
        _lib.call("rs_panel_lupp", S.data_ptr(), 64, Rp, 64, perm.data_ptr(), nc.data_ptr(),
                  ws.data_ptr(), st)
torch.cuda.synchronize()
print("done", what)
