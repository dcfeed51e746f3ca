"""Adaptive column ID on the cfg2 matrix (20000^2 fast decay, tau = 1e-8, b = 64,
device resident) with each sketch kind: wall time per run, rank, and the
sketch phase.  python tools/structured_adaptive.py [n]"""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import bench  # noqa: E402
import paper_2310_09417_b200 as rs  # noqa: E402


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 20000
    a = bench.gen_fast_decay_device(n, 1e-16, 0, torch.device("cuda")).T
    for kind in ("gaussian", "srtt", "sparsesign"):
        kw = {"zeta": 8} if kind == "sparsesign" else {}
        spec = rs.SketchSpec(kind, n, 64, **kw)
        for rep in range(2):
            torch.cuda.synchronize()
            t0 = time.time()
            res = rs.rand_lupp_adaptive(a, 64, 1e-8, spec, rs.RngStream(0))
            torch.cuda.synchronize()
            dt = time.time() - t0
            print(f"{kind:10s} n={n} rep {rep}: {dt * 1e3:.0f} ms, rank {res.rank}, status {res.status}", flush=True)


if __name__ == "__main__":
    main()
