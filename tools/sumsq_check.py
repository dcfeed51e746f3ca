import os, sys, numpy as np, torch
sys.path.insert(0, '/root/repo')
from paper_2310_09417_b200 import _lib, _device
lib = os.environ.get("RSKEL_LIB_PATH", "new")
rng = np.random.default_rng(0)
out = []
for R, w, ld in [(20000, 64, 64), (5000, 64, 80), (1234, 37, 37), (77, 300, 301), (3, 5, 5), (100000, 64, 64)]:
    X = torch.as_tensor(rng.standard_normal((R, ld)) * np.exp(rng.standard_normal((R, ld)))).cuda()
    o = torch.zeros(1, dtype=torch.float64, device="cuda")
    _lib.call("rs_sumsq", X.data_ptr(), ld, R, w, o.data_ptr(), _device.workspace().data_ptr(), _device.stream_handle())
    out.append(o.item().hex())
print(lib, out)
