"""Sketch GEMM efficiency vs block count batched into one product.
   PYTHONPATH=. python tools/sketch_width.py"""
import torch

from paper_2310_09417_b200 import _device, _lib

ws = _device.workspace()
st = _device.stream_handle()
n = 20000
a = torch.randn(n, n, dtype=torch.float64, device="cuda")
for nb in (1,):
    ell = 64 * nb
    om = torch.randn(n, ell, dtype=torch.float64, device="cuda")
    y = torch.empty(n, ell, dtype=torch.float64, device="cuda")
    f = lambda: _lib.call("rs_sketch_gemm", n, n, ell, a.data_ptr(), n, 1, om.data_ptr(), ell, y.data_ptr(), ell,
                          ws.data_ptr(), st)
    for _ in range(2):
        f()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(5):
        f()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    print(f"blocks {nb:2d} (N={ell}): {ms:.3f} ms, {2 * n * n * ell / ms / 1e9:.1f} TF/s, per block {ms / nb:.3f} ms")
