"""One Schur-block GEMM (S = Y[rest] - T Y[top]) at k = SCHUR_K for ncu.  python tools/schur_prof.py"""
import os
import sys

import torch

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
from paper_2310_09417_b200 import _device, _lib  # noqa: E402

m, b, k = 20000, 64, int(os.environ.get("SCHUR_K", 8000))
R = m - k
ws, st = _device.workspace().data_ptr(), _device.stream_handle()
Y = torch.randn(m, b, dtype=torch.float64, device="cuda")
perm = torch.randperm(m, device="cuda")
S = torch.empty(m, b, dtype=torch.float64, device="cuda")
T = torch.randn(R, k, dtype=torch.float64, device="cuda")
for _ in range(3):
    _lib.call("rs_schur_block", m, k, b, Y.data_ptr(), b, perm.data_ptr(), T.data_ptr(), k, S.data_ptr(), b, None, ws, st)
torch.cuda.synchronize()
print("ok")
