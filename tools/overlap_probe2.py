"""Could the sketch of block t+1 run beside the panel of block t if each took part of the GPU?
Sketch (20000^2 x 64) on a capped grid (OVL_SKETCH_LIB, e.g. 100 CTAs) and the panel on few
CTAs (OVL_PANEL_LIB, e.g. 250 rows per CTA -> 48 CTAs at R = 12000): alone and together on two
streams.   python tools/overlap_probe2.py"""
import ctypes
import os
import sys

import torch

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
sys.path.insert(0, os.path.join(REPO, "tools"))
from oz_check import slice_op  # noqa: E402
from paper_2310_09417_b200 import _device, _lib  # noqa: E402

sk = ctypes.CDLL(os.environ.get("OVL_SKETCH_LIB", _lib.LIB_PATH))
pn = ctypes.CDLL(os.environ.get("OVL_PANEL_LIB", _lib.LIB_PATH))
for lib in (sk, pn):
    lib.rs_oz_gemm.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_double,
                               ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p,
                               ctypes.c_int, ctypes.c_double, ctypes.c_void_p, ctypes.c_longlong, ctypes.c_void_p,
                               ctypes.c_longlong, ctypes.c_void_p, ctypes.c_void_p]
    lib.rs_panel_lupp.argtypes = [ctypes.c_void_p, ctypes.c_longlong, ctypes.c_int, ctypes.c_int, ctypes.c_void_p,
                                  ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]
n = 20000
A = torch.randn(n, n, dtype=torch.float64, device="cuda")
om = torch.randn(n, 64, dtype=torch.float64, device="cuda")
ad, ae, kc = slice_op(A, True, n, n, 8, 128)
bd, be, _ = slice_op(om, True, 64, n, 8, 64)
Y = torch.empty(n, 64, dtype=torch.float64, device="cuda")
R = int(os.environ.get("OVL_R", 12000))
S0 = torch.randn(R, 64, dtype=torch.float64, device="cuda")
Ss = [S0.clone() for _ in range(10)]
perm = torch.empty(R, dtype=torch.int64, device="cuda")
nc = torch.zeros(1, dtype=torch.int32, device="cuda")
ws1, ws2 = _device.workspace(1).data_ptr(), _device.workspace(2).data_ptr()
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def sketch(st):
    rc = sk.rs_oz_gemm(n, 64, n, kc, 0, 1.0, ad.data_ptr(), ae.data_ptr(), 8, bd.data_ptr(), be.data_ptr(), 8, 0.0,
                       None, 0, Y.data_ptr(), 64, ws1, st.cuda_stream)
    assert rc == 0


def panel(i, st):
    rc = pn.rs_panel_lupp(Ss[i].data_ptr(), 64, R, 64, perm.data_ptr(), nc.data_ptr(), ws2, st.cuda_stream)
    assert rc == 0


def timed(fn):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    fn()
    e1.record()
    torch.cuda.synchronize()
    return 1e3 * e0.elapsed_time(e1) / 10


cur = torch.cuda.current_stream()


def only_sketch():
    for _ in range(10):
        sketch(cur)


def only_panel():
    for i in range(10):
        panel(i, cur)


def both():
    for i in range(10):
        s1.wait_stream(cur)
        s2.wait_stream(cur)
        sketch(s1)
        panel(i, s2)
        cur.wait_stream(s1)
        cur.wait_stream(s2)


for f in (only_sketch, only_panel, both):
    f()
ts, tp, tb = timed(only_sketch), timed(only_panel), timed(both)
print(f"sketch {ts:.0f} us, panel R={R} {tp:.0f} us, sum {ts + tp:.0f} us, together {tb:.0f} us "
      f"({os.path.basename(os.environ.get('OVL_SKETCH_LIB', 'lib'))}, {os.path.basename(os.environ.get('OVL_PANEL_LIB', 'lib'))})",
      flush=True)
