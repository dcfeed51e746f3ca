"""SM clock and power while the tensor-core sketch GEMM runs back to back (cfg2 shape), and for
comparison while the DMMA Schur GEMM runs.  python tools/oz_clock.py"""
import os
import subprocess
import sys
import threading
import time

import torch

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
sys.path.insert(0, os.path.join(REPO, "tools"))
from oz_check import slice_op  # noqa: E402
from paper_2310_09417_b200 import _device, _lib  # noqa: E402

if os.environ.get("OZ_LIB"):
    _lib._lib = None
    _lib.load(os.environ["OZ_LIB"])

n = 20000
A = torch.randn(n, n, dtype=torch.float64, device="cuda")
om = torch.randn(n, 64, dtype=torch.float64, device="cuda")
ad, ae, kc = slice_op(A, True, n, n, 8, 128)
bd, be, _ = slice_op(om, True, 64, n, 8, 64)
Y = torch.empty(n, 64, dtype=torch.float64, device="cuda")
ws = _device.workspace().data_ptr()
st = _device.stream_handle()


def sample(out, stop):
    while not stop.is_set():
        r = subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm,power.draw,clocks_throttle_reasons.active",
                            "--format=csv,noheader,nounits"], capture_output=True, text=True)
        out.append(r.stdout.strip())
        time.sleep(0.05)


def run(label, fn, iters):
    fn(); torch.cuda.synchronize()
    out, stop = [], threading.Event()
    th = threading.Thread(target=sample, args=(out, stop)); th.start()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        fn()
    e1.record(); torch.cuda.synchronize()
    stop.set(); th.join()
    ms = e0.elapsed_time(e1) / iters
    mid = out[len(out) // 4: 3 * len(out) // 4] or out
    print(f"{label}: {ms:.3f} ms/iter; nvidia-smi (sm MHz, W, reasons) mid-run: {mid[:: max(1, len(mid) // 8)]}", flush=True)


def oz():
    _lib.call("rs_oz_gemm", n, 64, n, kc, 0, 1.0, ad.data_ptr(), ae.data_ptr(), 8, bd.data_ptr(), be.data_ptr(), 8,
              0.0, None, 0, Y.data_ptr(), 64, ws, st)


zd = torch.zeros_like(ad)
def oz_zero():
    _lib.call("rs_oz_gemm", n, 64, n, kc, 0, 1.0, zd.data_ptr(), ae.data_ptr(), 8, bd.data_ptr(), be.data_ptr(), 8,
              0.0, None, 0, Y.data_ptr(), 64, ws, st)


run("oz_gemm random digits", oz, 3000)
run("oz_gemm zero A digits", oz_zero, 3000)
