"""One adaptive column ID at the cfg2 shape inside an NVTX range "step" (after a warm-up call), for
ncu launch lists:  ncu --nvtx --nvtx-include "step/" --metrics gpu__time_duration.sum --csv \
   --clock-control none python tools/prof_step.py"""
import os
import sys

import torch

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
import paper_2310_09417_b200 as rs  # noqa: E402
from bench import gen_fast_decay_device  # noqa: E402

n = int(os.environ.get("PROF_N", 20000))
a = gen_fast_decay_device(n, 1e-16, 0, torch.device("cuda", 0))
spec = rs.SketchSpec("gaussian", n, 64)
rs.rand_lupp_adaptive(a.T, 64, 1e-8, spec, rs.RngStream(0))
torch.cuda.synchronize()
torch.cuda.nvtx.range_push("step")
res = rs.rand_lupp_adaptive(a.T, 64, 1e-8, spec, rs.RngStream(0))
torch.cuda.synchronize()
torch.cuda.nvtx.range_pop()
print("rank", res.rank)
