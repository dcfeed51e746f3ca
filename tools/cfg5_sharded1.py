"""cfg5 through the column-sharded loop at one rank (the N > 1 code path at
full scale).   PYTHONPATH=. python tools/cfg5_sharded1.py"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2310_09417_b200 as rs  # noqa: E402
from bench_configs import algo_flops, gen_fast_decay_hadamard  # noqa: E402
from paper_2310_09417_b200.sharded import rand_lupp_adaptive_sharded  # noqa: E402

n, b, tau = int(os.environ.get("CFG5_N", 65536)), 64, 1e-8
a = gen_fast_decay_hadamard(n, 1e-16, 0)
spec = rs.SketchSpec("gaussian", n, b)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
torch.cuda.synchronize()
e0.record()
res = rand_lupp_adaptive_sharded(a.T, b, tau, spec, rs.RngStream(0))
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1)
print(f"cfg5 sharded loop, 1 rank: {ms / 1e3:.2f} s, rank {res.rank}, status {res.status}, "
      f"blocks {len(res.trace) + 1}, {algo_flops(n, n, res.rank, b) / ms / 1e9:.1f} TF/s", flush=True)
