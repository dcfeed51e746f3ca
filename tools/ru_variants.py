import os, sys, torch
import paper_2310_09417_b200._lib as L
L._lib = None
L.load(os.path.join(os.path.dirname(__file__), sys.argv[1]))
from paper_2310_09417_b200 import _device, _lib
exec(open(os.path.join(os.path.dirname(__file__), "bench_kernels.py")).read().split("def bench_panel")[0])
st = _device.stream_handle()
n = 20000
for k in (2000, 7000, 14000):
    R = n - k
    T = torch.randn(R, k, dtype=torch.float64, device="cuda")
    sub = torch.randperm(R, device="cuda")
    Tn = torch.empty((R - 64) * (k + 64), dtype=torch.float64, device="cuda")
    What = torch.randn(R - 64, 64, dtype=torch.float64, device="cuda")
    ms = timeit(lambda: _lib.call("rs_rank_update", R - 64, k, 64, What.data_ptr(), 64, T.data_ptr(), k,
                                  sub.data_ptr(), T.data_ptr(), k, sub.data_ptr() + 8 * 64, Tn.data_ptr(), k, st), reps=10)
    Tref = T[sub[64:]] - What @ T[sub[:64]]
    err = float((Tn[: (R - 64) * k].view(R - 64, k) - Tref).abs().max())
    print(f"{sys.argv[1]} k={k}: {ms:.3f} ms {2*(R-64)*64*k/ms/1e9:.1f} TF/s err {err}")
