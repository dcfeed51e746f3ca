"""Per-launch panel times (CUDA events around each of 30 back-to-back launches).
   python tools/panel_launches.py [R ...]"""
import os
import sys

import torch

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
from paper_2310_09417_b200 import _device, _lib  # noqa: E402

if os.environ.get("PANEL_LIB"):  # an experiment build instead of the library
    _lib._lib = None
    _lib.load(os.environ["PANEL_LIB"])

ws, st = _device.workspace().data_ptr(), _device.stream_handle()
for R in [int(x) for x in (sys.argv[1:] or ["2000", "4096", "16000"])]:
    S0 = torch.randn(R, 64, dtype=torch.float64, device="cuda")
    Ss = [S0.clone() for _ in range(30)]
    perm = torch.empty(R, dtype=torch.int64, device="cuda")
    nc = torch.zeros(1, dtype=torch.int32, device="cuda")
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(31)]
    _lib.call("rs_panel_lupp", S0.clone().data_ptr(), 64, R, 64, perm.data_ptr(), nc.data_ptr(), ws, st)
    torch.cuda.synchronize()
    ev[0].record()
    for i, X in enumerate(Ss):
        _lib.call("rs_panel_lupp", X.data_ptr(), 64, R, 64, perm.data_ptr(), nc.data_ptr(), ws, st)
        ev[i + 1].record()
    torch.cuda.synchronize()
    t = [1e3 * ev[i].elapsed_time(ev[i + 1]) for i in range(30)]
    print(f"{os.path.basename(os.environ.get('PANEL_LIB', 'librskel.so'))} R={R}: " + " ".join(f"{x:.0f}" for x in t) + f"  (us per launch; median {sorted(t)[15]:.0f})", flush=True)
