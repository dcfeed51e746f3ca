"""Which fp64 formulation parts from the oracle first on the cfg2 recipe: the T-form engine of
`rand_lupp_adaptive` (S = Y[rest] - T Y[top], T updated in place) or the device L-form
resumable API (`adaptive_init` / `adaptive_step`: S = PY[k:] - L2 L1^-1 PY[:k], the
reference's `skeleton.py:317-323` formulation, every product on the same device kernels).

Prints the common pivot prefixes T/oracle, L/oracle and T/L.  If the L-form follows the
oracle further than the T-form, T drift is the extra rounding; if both part where the oracle
has a near tie, the tie is inherent to fp64.  Test infrastructure (the oracle is the checker).

  python tools/lform_vs_tform.py --n 6000
"""
import argparse
import json
import os
import sys

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
sys.path.insert(0, os.path.join(REPO, "oracle"))


def prefix(a, b):
    n = min(len(a), len(b))
    d = np.nonzero(np.asarray(a[:n]) != np.asarray(b[:n]))[0]
    return n if d.size == 0 else int(d[0])


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=6000)
    ap.add_argument("--b", type=int, default=64)
    ap.add_argument("--tau", type=float, default=1e-8)
    ap.add_argument("--out", default=None)
    args = ap.parse_args()

    import torch
    from threadpoolctl import threadpool_limits

    import bench
    import paper_2310_09417_b200 as rs
    import randskel_oracle as orc

    n, b, tau = args.n, args.b, args.tau
    dev = torch.device("cuda", 0)
    a = bench.gen_fast_decay_device(n, 1e-16, 0, dev)
    at = a.T.contiguous()
    spec = rs.SketchSpec("gaussian", n, b)
    res = rs.rand_lupp_adaptive(at, b, tau, spec, rs.RngStream(0))
    t_idx = res.row_idx.cpu().numpy()

    st = rs.adaptive_init(at, b, spec, rs.RngStream(0))
    l_trace = []
    while st.rank + b <= n:
        e, nxt = rs.adaptive_step(st, at, spec)
        l_trace.append((st.rank, e))
        if e <= tau:
            break
        st = nxt
    l_idx = st.perm[:st.rank].cpu().numpy() if hasattr(st.perm, "cpu") else np.asarray(st.perm[:st.rank])

    with threadpool_limits(limits=os.cpu_count() or 1):
        ref = orc.rand_lupp_adaptive(a.cpu().numpy().T, b, tau, 0, 0, want_w=False)
    r_idx = np.asarray(ref["row_idx"])
    out = {"n": n, "b": b, "tau": tau,
           "rank": {"tform": int(res.rank), "lform": int(st.rank), "oracle": int(ref["rank"])},
           "prefix": {"tform_oracle": prefix(t_idx, r_idx), "lform_oracle": prefix(l_idx, r_idx),
                      "tform_lform": prefix(t_idx, l_idx)}}
    line = json.dumps(out)
    print(line, flush=True)
    if args.out:
        with open(args.out, "w") as f:
            f.write(line + "\n")


if __name__ == "__main__":
    main()
