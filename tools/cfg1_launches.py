"""One cfg1 column ID (4096^2, k = 256, device input) inside an NVTX range for an ncu launch list.
   ncu --nvtx --nvtx-include "cfg1/" --metrics gpu__time_duration.sum --csv python tools/cfg1_launches.py"""
import os
import sys

import torch

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
import paper_2310_09417_b200 as rs  # noqa: E402
from bench_configs import gen_fast_decay_device  # noqa: E402

n, k = 4096, 256
a = gen_fast_decay_device(n, 1e-16, 0, "cuda")
spec = rs.SketchSpec("gaussian", n, k)
for _ in range(2):
    rs.column_id(a, k, spec, rs.RngStream(0))
torch.cuda.synchronize()
torch.cuda.nvtx.range_push("cfg1")
rs.column_id(a, k, spec, rs.RngStream(0))
torch.cuda.synchronize()
torch.cuda.nvtx.range_pop()
