import ctypes, os
import numpy as np
import torch
import paper_2310_09417_b200._lib as L
lib = L.load(os.path.join(os.path.dirname(__file__), "librskel_prof.so"))
lib.rs_panel_prof.argtypes = [ctypes.c_void_p]
from paper_2310_09417_b200 import _device
ws = _device.workspace()
for R in (2000, 20000):
    s0 = torch.randn(R, 64, dtype=torch.float64, device="cuda"); S = s0.clone()
    perm = torch.empty(R, dtype=torch.int64, device="cuda"); nc = torch.empty(1, dtype=torch.int32, device="cuda")
    out = np.zeros(2 * 66 * 160, dtype=np.uint64)
    for it in range(3):
        S.copy_(s0)
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        lib.rs_panel_lupp(S.data_ptr(), 64, R, 64, perm.data_ptr(), nc.data_ptr(), ws.data_ptr(), _device.stream_handle())
        e1.record()
        torch.cuda.synchronize()
    lib.rs_panel_prof(out.ctypes.data)
    G = min(148, (R + 127) // 128)
    pub, seen = [out[i*66*160:(i+1)*66*160].reshape(66, 160)[:, :G].astype(np.int64) for i in range(2)]
    t0 = pub[64].min()
    print(f"R={R} G={G} event ms {e0.elapsed_time(e1):.3f}; kernel start spread {pub[64].max()-t0} ns; first pub {pub[0].min()-t0}; end {pub[65].max()-t0} ns")
    steps = np.diff(np.median(pub[:64], axis=1))
    print("  step ns (median over CTAs):", steps.astype(int).tolist())
    print("  pub spread per step:", (pub[:64].max(1) - pub[:64].min(1)).astype(int).tolist()[:16])
    print("  seen - lastpub (min,max):", [(int(seen[j].min()-pub[j].max()), int(seen[j].max()-pub[j].max())) for j in range(0, 64, 8)])
