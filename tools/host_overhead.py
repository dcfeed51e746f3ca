"""Host-side cost of enqueueing the library's kernels (wall time of the C call, no sync), e.g.
the cooperative panel launch.  python tools/host_overhead.py"""
import os
import sys
import time

import torch

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
from paper_2310_09417_b200 import _device, _lib  # noqa: E402

ws, st = _device.workspace().data_ptr(), _device.stream_handle()
for R in (2000, 6000, 16000):
    S = torch.randn(R, 64, dtype=torch.float64, device="cuda")
    perm = torch.empty(R, dtype=torch.int64, device="cuda")
    nc = torch.zeros(1, dtype=torch.int32, device="cuda")
    _lib.call("rs_panel_lupp", S.data_ptr(), 64, R, 64, perm.data_ptr(), nc.data_ptr(), ws, st)
    torch.cuda.synchronize()
    n = 50
    t0 = time.perf_counter()
    for _ in range(n):
        _lib.call("rs_panel_lupp", S.data_ptr(), 64, R, 64, perm.data_ptr(), nc.data_ptr(), ws, st)
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        _lib.call("rs_panel_lupp", S.data_ptr(), 64, R, 64, perm.data_ptr(), nc.data_ptr(), ws, st)
    e1.record()
    torch.cuda.synchronize()
    print(f"panel R={R}: host enqueue {1e6 * (t1 - t0) / n:.1f} us/call, wall incl. drain {1e6 * (t2 - t0) / n:.1f} us/call, "
          f"device events {1e3 * e0.elapsed_time(e1) / n:.1f} us/call", flush=True)
