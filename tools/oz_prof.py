"""One Ozaki sketch GEMM at the cfg2 shape (20000^2 x 64) for ncu.  PYTHONPATH=. python tools/oz_prof.py"""
import os
import sys

import torch

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
sys.path.insert(0, os.path.join(REPO, "tools"))
from oz_check import slice_op  # noqa: E402
from paper_2310_09417_b200 import _device, _lib  # noqa: E402

if os.environ.get("OZ_LIB"):
    _lib._lib = None
    _lib.load(os.environ["OZ_LIB"])

n = int(os.environ.get("OZ_N", 20000))
SA = int(os.environ.get("OZ_SA", 8))
A = torch.randn(n, n, dtype=torch.float64, device="cuda")
om = torch.randn(n, 64, dtype=torch.float64, device="cuda")
ad, ae, kc = slice_op(A, True, n, n, SA, 128)
bd, be, _ = slice_op(om, True, 64, n, 8, 64)
Y = torch.empty(n, 64, dtype=torch.float64, device="cuda")
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for rep in range(3):
    e0.record()
    _lib.call("rs_oz_gemm", n, 64, n, kc, 0, 1.0, ad.data_ptr(), ae.data_ptr(), SA, bd.data_ptr(), be.data_ptr(), 8,
              0.0, None, 0, Y.data_ptr(), 64, _device.workspace().data_ptr(), _device.stream_handle())
    e1.record()
    torch.cuda.synchronize()
print(f"ok {os.environ.get('OZ_LIB', 'librskel')} SA={SA}: {e0.elapsed_time(e1):.3f} ms")
