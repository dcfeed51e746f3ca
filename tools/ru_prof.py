"""One rank update T' = T[Q] - W_hat T[P] (the absorb step) at k = RU_K for ncu.  python tools/ru_prof.py"""
import os
import sys

import torch

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
from paper_2310_09417_b200 import _device, _lib  # noqa: E402

if os.environ.get("RU_LIB"):  # an experiment build instead of the library
    _lib._lib = None
    _lib.load(os.environ["RU_LIB"])

m, b, k = 20000, 64, int(os.environ.get("RU_K", 8000))
R = m - k - b
st = _device.stream_handle()
T = torch.randn(m - k, k, dtype=torch.float64, device="cuda")
Tn = torch.empty(R, k + b, dtype=torch.float64, device="cuda")
sub = torch.randperm(m - k, device="cuda")
for _ in range(3):
    _lib.call("rs_rank_update", R, k, b, Tn.data_ptr() + 8 * k, k + b, T.data_ptr(), k, sub.data_ptr(),
              T.data_ptr(), k, sub[b:].data_ptr(), Tn.data_ptr(), k + b, st)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10):
    _lib.call("rs_rank_update", R, k, b, Tn.data_ptr() + 8 * k, k + b, T.data_ptr(), k, sub.data_ptr(),
              T.data_ptr(), k, sub[b:].data_ptr(), Tn.data_ptr(), k + b, st)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 10
print(f"{os.path.basename(os.environ.get('RU_LIB', 'librskel.so'))} rank update R={R} k={k}: {ms:.3f} ms, {2 * R * k * b / ms / 1e9:.1f} TF/s, {16 * R * k / ms / 1e6:.0f} GB/s")
