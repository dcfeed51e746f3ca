"""Per-CTA publish / winner-known times (globaltimer, ns) of the panel exchange.
Needs tools/librskel_prof.so (-DRS_PANEL_PROBE_ON).  PYTHONPATH=. python tools/panel_skew.py"""
import ctypes
import os

import numpy as np
import torch

import paper_2310_09417_b200._lib as L

lib = L.load(os.path.join(os.path.dirname(__file__), os.environ.get("PROF_LIB", "librskel_prof.so")))
lib.rs_panel_gt.argtypes = [ctypes.c_void_p]
from paper_2310_09417_b200 import _device  # noqa: E402

ws = _device.workspace()
for R in (2000, 20000):
    s0 = torch.randn(R, 64, dtype=torch.float64, device="cuda")
    S = s0.clone()
    perm = torch.empty(R, dtype=torch.int64, device="cuda")
    nc = torch.empty(1, dtype=torch.int32, device="cuda")
    for _ in range(3):
        S.copy_(s0)
        lib.rs_panel_lupp(S.data_ptr(), 64, R, 64, perm.data_ptr(), nc.data_ptr(), ws.data_ptr(),
                          _device.stream_handle())
        torch.cuda.synchronize()
    out = np.zeros(6 * 64 * 256, dtype=np.uint64)
    lib.rs_panel_gt(out.ctypes.data)
    t = out.reshape(6, 64, 256).astype(np.int64)
    G = int((t[0, 10] > 0).sum())
    for j in (10, 11, 30):
        st, pub, known = t[0, j, :G], t[1, j, :G], t[2, j, :G]
        base = st.min()
        print(f"R={R} G={G} col {j}: start spread {st.max() - st.min()} ns, publish spread "
              f"{pub.max() - pub.min()} ns (last CTA {int(pub.argmax())}), known - last publish: "
              f"min {known.min() - pub.max()} max {known.max() - pub.max()} ns, step {t[0, j + 1, :G].min() - base} ns")
        print("   publish offsets (ns):", (pub - base)[:16].tolist())
        print("   poll passes (lane 0):", t[3, j, :G][:16].tolist())
        print("   issue - publish (ns):", (t[4, j, :G] - pub)[:16].tolist())
        print("   load latency (ns):", (t[5, j, :G] - t[4, j, :G])[:16].tolist())
