"""Panel LUPP time (R x 64) for the library build and experiment builds.  python tools/panel_time.py [lib.so ...]"""
import os
import sys

import torch

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
from paper_2310_09417_b200 import _device, _lib  # noqa: E402

for path in sys.argv[1:] or [""]:
    if path:
        _lib._lib = None
        _lib.load(path)
    ws, st = _device.workspace().data_ptr(), _device.stream_handle()
    row = []
    for R in [int(x) for x in os.environ.get("PANEL_RS", "2000,6000,10000,16000,20000,40000,65000").split(",")]:
        S0 = torch.randn(R, 64, dtype=torch.float64, device="cuda")
        S = S0.clone()
        perm = torch.empty(R, dtype=torch.int64, device="cuda")
        nc = torch.zeros(1, dtype=torch.int32, device="cuda")
        Ss = [S0.clone() for _ in range(int(os.environ.get("PANEL_REPS", 20)))]
        _lib.call("rs_panel_lupp", S.data_ptr(), 64, R, 64, perm.data_ptr(), nc.data_ptr(), ws, st)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for X in Ss:  # back to back: clocks stay up, launch gaps hidden
            _lib.call("rs_panel_lupp", X.data_ptr(), 64, R, 64, perm.data_ptr(), nc.data_ptr(), ws, st)
        e1.record()
        torch.cuda.synchronize()
        row.append(f"R={R}:{1e3 * e0.elapsed_time(e1) / len(Ss):.0f}us")
        del Ss
    print(path or "librskel.so", " ".join(row), flush=True)
