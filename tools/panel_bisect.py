"""Per-column panel cost (R = 2000 / 20000, w = 64) for experiment builds.
   PYTHONPATH=. python tools/panel_bisect.py librskel_exp7.so ..."""
import os
import sys

import torch

import paper_2310_09417_b200._lib as L

for name in sys.argv[1:]:
    L._lib = None
    lib = L.load(os.path.join(os.path.dirname(os.path.abspath(__file__)), name) if name != "prod" else L.LIB_PATH)
    from paper_2310_09417_b200 import _device

    ws = _device.workspace()
    res = []
    for R in (2000, 20000):
        s0 = torch.randn(R, 64, dtype=torch.float64, device="cuda")
        S = s0.clone()
        perm = torch.empty(R, dtype=torch.int64, device="cuda")
        nc = torch.empty(1, dtype=torch.int32, device="cuda")
        ts = {}
        for w in (1, 64):
            for _ in range(3):
                S.copy_(s0)
                lib.rs_panel_lupp(S.data_ptr(), 64, R, w, perm.data_ptr(), nc.data_ptr(), ws.data_ptr(),
                                  _device.stream_handle())
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            tot = 0.0
            for _ in range(10):
                S.copy_(s0)
                e0.record()
                lib.rs_panel_lupp(S.data_ptr(), 64, R, w, perm.data_ptr(), nc.data_ptr(), ws.data_ptr(),
                                  _device.stream_handle())
                e1.record()
                torch.cuda.synchronize()
                tot += e0.elapsed_time(e1)
            ts[w] = tot / 10
        res.append(f"R={R}: w1 {1e3 * ts[1]:.1f} us, per column {1e3 * (ts[64] - ts[1]) / 63:.2f} us")
    print(name, "|", "; ".join(res), flush=True)
