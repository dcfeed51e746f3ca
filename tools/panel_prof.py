"""Per-phase panel timeline (clock64 of thread 0 in CTAs 0/1, kept in shared
memory during the run).  Needs tools/librskel_prof.so built with
-DRS_PANEL_PROBE_ON.   PYTHONPATH=. python tools/panel_prof.py"""
import ctypes
import os

import numpy as np
import torch

import paper_2310_09417_b200._lib as L

lib = L.load(os.path.join(os.path.dirname(__file__), os.environ.get("PROF_LIB", "librskel_prof.so")))
lib.rs_panel_probe.argtypes = [ctypes.c_void_p]
from paper_2310_09417_b200 import _device  # noqa: E402

ws = _device.workspace()
names = {1: "published", 2: "winner known", 3: "U row loaded", 5: "after sync", 6: "early done",
         4: "block_best done", 7: "end"}
for R in (2000, 6000, 20000, 65472):
    s0 = torch.randn(R, 64, dtype=torch.float64, device="cuda")
    S = s0.clone()
    perm = torch.empty(R, dtype=torch.int64, device="cuda")
    nc = torch.empty(1, dtype=torch.int32, device="cuda")
    out = np.zeros(2 * 8 * 64, dtype=np.uint64)
    for it in range(3):
        S.copy_(s0)
        torch.cuda.synchronize()
        lib.rs_panel_lupp(S.data_ptr(), 64, R, 64, perm.data_ptr(), nc.data_ptr(), ws.data_ptr(),
                          _device.stream_handle())
        torch.cuda.synchronize()
    lib.rs_panel_probe(out.ctypes.data)
    t = out.reshape(2, 8, 64).astype(np.int64)
    for c in (0, 1):
        d = {names[k]: int(np.median(t[c, k, 2:62] - t[c, 0, 2:62])) for k in sorted(names)}
        print(f"R={R:6d} cta{c} step {int(np.median(np.diff(t[c, 0, 2:62])))} cycles:", d)
