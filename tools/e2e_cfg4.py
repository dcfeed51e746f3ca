"""cfg4 end-to-end column_id time, streamed vs plain H2D.   PYTHONPATH=. python tools/e2e_cfg4.py"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle"))
import paper_2310_09417_b200 as rs  # noqa: E402
import randskel_oracle as orc  # noqa: E402

n, k = 16384, 1024
a = orc.gen_kahan(n, 0.99)
spec = rs.SketchSpec("gaussian", n, k)
for mode in ("0", "1", "0", "1"):
    os.environ["RSKEL_PRESKETCH"] = mode
    ts = []
    for _ in range(3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        r = rs.column_id(a, k, spec, rs.RngStream(0))
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    print(f"RSKEL_PRESKETCH={mode}: e2e {[round(1e3 * t, 1) for t in ts]} ms", flush=True)
