"""Skeleton / Schur gathers: achieved HBM GB/s (read + write bytes / CUDA-event time, 20 launches
back to back) at the path's shapes.  python tools/gather_prof.py   (ncu: GATHER_REPS=1)"""
import os
import sys

import torch

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
from paper_2310_09417_b200 import _device, _lib  # noqa: E402

reps = int(os.environ.get("GATHER_REPS", 20))
dev = torch.device("cuda")
st = _device.stream_handle()
g = torch.Generator(device="cpu").manual_seed(0)
A = torch.randn(32768, 16384, dtype=torch.float64, device=dev)           # cfg3-sized a (row-major)
Y = torch.randn(20000, 64, dtype=torch.float64, device=dev)              # one sketch block
perm = torch.randperm(20000, generator=g).to(dev)
I = torch.randperm(32768, generator=g)[:256].to(dev)
J = torch.randperm(16384, generator=g)[:256].to(dev)
cases = []
S = torch.empty(20000, 64, dtype=torch.float64, device=dev)
cases.append(("Y[perm] 20000x64 (Schur block rows)", lambda: _lib.call(
    "rs_gather_rows", Y.data_ptr(), 64, perm.data_ptr(), 20000, 64, S.data_ptr(), 64, st), 2 * S.numel() * 8))
R = torch.empty(256, 16384, dtype=torch.float64, device=dev)
cases.append(("R = a[I, :] 256x16384 of 32768x16384 row-major", lambda: _lib.call(
    "rs_gather2d", A.data_ptr(), 16384, 1, I.data_ptr(), 256, None, 16384, R.data_ptr(), 16384, st), 2 * R.numel() * 8))
C = torch.empty(32768, 256, dtype=torch.float64, device=dev)
cases.append(("C = a[:, J] 32768x256 of row-major a (scattered 8-byte columns)", lambda: _lib.call(
    "rs_gather2d", A.data_ptr(), 16384, 1, None, 32768, J.data_ptr(), 256, C.data_ptr(), 256, st), 2 * C.numel() * 8))
# column-major a: the same logical matrix stored transposed (a = At.T), rs = 1, cs = 32768
At = torch.randn(16384, 32768, dtype=torch.float64, device=dev)
cases.append(("C = a[:, J] 32768x256 of column-major a (tiled transpose)", lambda: _lib.call(
    "rs_gather2d", At.data_ptr(), 1, 32768, None, 32768, J.data_ptr(), 256, C.data_ptr(), 256, st), 2 * C.numel() * 8))
for name, fn, nbytes in cases:
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    us = 1e3 * e0.elapsed_time(e1) / reps
    print(f"{name}: {us:.1f} us, {nbytes / us / 1e3:.0f} GB/s (read + write)", flush=True)
