"""Panel time vs panel width: separates the fixed cost (launch, smem fill,
write-back) from the per-column exchange.   PYTHONPATH=. python tools/panel_fixed.py"""
import torch

from paper_2310_09417_b200 import _device, _lib

ws = _device.workspace()


def timeit(fn, reps=20):
    for _ in range(3):
        fn()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


for R in (2000, 20000):
    s0 = torch.randn(R, 64, dtype=torch.float64, device="cuda")
    S = s0.clone()
    perm = torch.empty(R, dtype=torch.int64, device="cuda")
    nc = torch.empty(1, dtype=torch.int32, device="cuda")
    copy = timeit(lambda: S.copy_(s0))
    out = []
    for w in (1, 2, 8, 32, 64):
        ms = timeit(lambda: (S.copy_(s0), _lib.call("rs_panel_lupp", S.data_ptr(), 64, R, w, perm.data_ptr(),
                                                     nc.data_ptr(), ws.data_ptr(), _device.stream_handle())))
        out.append(f"w={w}: {1e3 * (ms - copy):.1f} us")
    print(f"R={R}: " + ", ".join(out))
