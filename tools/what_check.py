"""rs_what (W_hat rows by substitution) on fixed random inputs: prints a digest of every output
and the time, so two builds can be compared bit for bit (RSKEL_LIB_PATH=<variant .so>)."""
import hashlib
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
from paper_2310_09417_b200 import _device, _lib  # noqa: E402

rng = np.random.default_rng(0)
dig = []
for R, nc, lds in [(20000, 64, 64), (15000, 63, 64), (7, 5, 9), (1, 1, 1), (3000, 64, 70), (129, 33, 40)]:
    m = R + nc
    S = torch.as_tensor(rng.standard_normal((m, lds))).cuda()
    sub = torch.as_tensor(rng.permutation(m)[:nc].astype(np.int64)).cuda()
    ridx = torch.as_tensor(rng.permutation(m)[:R].astype(np.int64)).cuda()
    out = torch.zeros(R, nc, dtype=torch.float64, device="cuda")
    args = (S.data_ptr(), lds, sub.data_ptr(), nc, ridx.data_ptr(), R, out.data_ptr(), nc, _device.stream_handle())
    _lib.call("rs_what", *args)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        _lib.call("rs_what", *args)
    e1.record()
    torch.cuda.synchronize()
    dig.append((R, nc, hashlib.sha1(out.cpu().numpy().tobytes()).hexdigest()[:12], round(e0.elapsed_time(e1) / 20 * 1e3, 1)))
print(os.environ.get("RSKEL_LIB_PATH", "librskel.so"), dig)
