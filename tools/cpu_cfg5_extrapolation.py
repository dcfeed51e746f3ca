"""the reference algorithm on the host cores at 16384^2 and 32768^2 (cfg5 recipe:
randomized-Hadamard fast decay, b = 64, tau = 1e-8), next to the GPU on the same matrices, and the
n-exponent extrapolation to 65536^2.  The oracle port (numpy/OpenBLAS, all host cores) is timed;
the GPU result is compared with it (rank, common pivot prefix).  Test infrastructure.

  python tools/cpu_cfg5_extrapolation.py [--n 16384 32768]
"""
import argparse
import json
import math
import os
import sys
import time

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
sys.path.insert(0, os.path.join(REPO, "oracle"))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, nargs="+", default=[16384, 32768])
    args = ap.parse_args()
    import torch
    from threadpoolctl import threadpool_limits

    import paper_2310_09417_b200 as rs
    import randskel_oracle as orc
    from bench import algo_flops

    cores = os.cpu_count()
    pts = []
    for n in args.n:
        a, _ = rs.gen_fast_decay_hadamard(n, 1e-16, rs.RngStream(0).child(1 << 41))
        spec = rs.SketchSpec("gaussian", n, 64)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        res = rs.rand_lupp_adaptive(a.T, 64, 1e-8, spec, rs.RngStream(0))
        torch.cuda.synchronize()
        gpu_s = time.perf_counter() - t0
        t0 = time.perf_counter()
        res = rs.rand_lupp_adaptive(a.T, 64, 1e-8, spec, rs.RngStream(0))
        torch.cuda.synchronize()
        gpu_s = min(gpu_s, time.perf_counter() - t0)
        g_idx = res.row_idx.cpu().numpy()
        h = a.cpu().numpy()
        del a
        torch.cuda.empty_cache()
        with threadpool_limits(limits=cores):
            t0 = time.perf_counter()
            ref = orc.rand_lupp_adaptive(np.ascontiguousarray(h.T), 64, 1e-8, 0, 0, want_w=False)
            cpu_s = time.perf_counter() - t0
        r_idx = np.asarray(ref["row_idx"])
        m = min(len(g_idx), len(r_idx))
        d = np.nonzero(g_idx[:m] != r_idx[:m])[0]
        f = algo_flops(n, n, ref["rank"], 64)
        line = {"n": n, "cpu_s": cpu_s, "cpu_cores": cores, "cpu_tflops": f / cpu_s / 1e12, "gpu_s": gpu_s,
                "rank_cpu": int(ref["rank"]), "rank_gpu": int(res.rank), "status": [ref["status"], res.status],
                "common_pivot_prefix": int(m if d.size == 0 else d[0]), "speedup": cpu_s / gpu_s}
        pts.append(line)
        print(json.dumps(line), flush=True)
        del h
    if len(pts) >= 2:
        (n1, t1), (n2, t2) = (pts[-2]["n"], pts[-2]["cpu_s"]), (pts[-1]["n"], pts[-1]["cpu_s"])
        p = math.log(t2 / t1) / math.log(n2 / n1)
        print(json.dumps({"extrapolation": "cpu_s(65536) = cpu_s(n2) * (65536/n2)^p", "p": p,
                          "cpu_s_65536_est": t2 * (65536 / n2) ** p}), flush=True)


if __name__ == "__main__":
    main()
