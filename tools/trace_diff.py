"""Per-block e_schur difference, CUDA path vs the oracle, on the cfg2 recipe at n
(tests/test_gpu_cfg2_scale.py's matrix).  Test infrastructure (the oracle is the checker).

  python tools/trace_diff.py --n 6000
"""
import argparse
import os
import sys

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
sys.path.insert(0, os.path.join(REPO, "oracle"))
sys.path.insert(0, os.path.join(REPO, "tests"))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=6000)
    args = ap.parse_args()
    import torch
    from threadpoolctl import threadpool_limits

    import paper_2310_09417_b200 as rs
    import randskel_oracle as orc
    from test_gpu_cfg2_scale import _gen_fast_decay_device

    n, b, tau = args.n, 64, 1e-8
    a = _gen_fast_decay_device(n, 1e-16, 0, torch.device("cuda", 0))
    res = rs.rand_lupp_adaptive(a.T, b, tau, rs.SketchSpec("gaussian", n, b), rs.RngStream(0))
    with threadpool_limits(limits=os.cpu_count() or 1):
        ref = orc.rand_lupp_adaptive(a.cpu().numpy().T, b, tau, 0, 0, want_w=False)
    na = float(torch.linalg.norm(a))
    g = res.row_idx.cpu().numpy()
    r = np.asarray(ref["row_idx"])
    m = min(len(g), len(r))
    d = np.nonzero(g[:m] != r[:m])[0]
    p0 = m if d.size == 0 else int(d[0])
    print(f"rank {res.rank}/{ref['rank']} prefix {p0} ||A|| {na:.6e}")
    for (k, e), (k0, e0) in zip([(x.k, x.e_schur) for x in res.trace], ref["trace"]):
        flag = "" if k <= p0 else " (after parting)"
        print(f"k={k:5d} e/||A||={e0 / na:.3e} |de|/||A||={abs(e - e0) / na:.3e} rel={abs(e - e0) / e0:.3e}{flag}")


if __name__ == "__main__":
    main()
