"""Full-size cfg2 parity: the CUDA path against the oracle port on the SAME matrix.

BASELINE.json configs[1]: rand_lupp_adaptive(A.T, b=64, tau=1e-8 (absolute), Gaussian,
RngStream(0)) on the 20000^2 fp64 fast-decay matrix bench.py times (beta=1e-16, Haar bases
generated on the device).  The oracle (oracle/randskel_oracle.py, numpy/OpenBLAS on all
host cores; it restates `skeleton.py:391-460` and is pinned against the reference's golden
vectors) runs the whole adaptive loop on the host copy of the same A -- several minutes.

Reports rank / status / trace length, the common prefix and set overlap of row_idx, the
largest trace difference relative to ||A||_F, the e_schur values around tau, the entrywise
W difference and both residuals ||A.T - W A.T[I]||_F / ||A||_F.  Test infrastructure: the
oracle is the checker here, never the thing measured.

  python tools/cfg2_full_parity.py --n 20000 --out gpurun_out/cfg2_full_parity.json
"""
import argparse
import json
import os
import sys
import time

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
sys.path.insert(0, os.path.join(REPO, "oracle"))


def host(x):
    import torch

    return x.cpu().numpy() if isinstance(x, torch.Tensor) else np.asarray(x)


def prefix(a, b):
    n = min(len(a), len(b))
    d = np.nonzero(a[:n] != b[:n])[0]
    return n if d.size == 0 else int(d[0])


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=20000)
    ap.add_argument("--b", type=int, default=64)
    ap.add_argument("--tau", type=float, default=1e-8)
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--out", default=None)
    ap.add_argument("--rowmajor", action="store_true", help="pass A.T as a row-major copy, not the column-major view")
    args = ap.parse_args()

    import torch
    from threadpoolctl import threadpool_limits

    import bench
    import paper_2310_09417_b200 as rs
    import randskel_oracle as orc

    dev = torch.device("cuda", 0)
    n, b, tau = args.n, args.b, args.tau
    a = bench.gen_fast_decay_device(n, 1e-16, args.seed, dev)
    norm_a = float(torch.linalg.norm(a))
    spec = rs.SketchSpec("gaussian", n, b)

    torch.cuda.synchronize()
    t0 = time.perf_counter()
    at_in = a.T.contiguous() if args.rowmajor else a.T
    res = rs.rand_lupp_adaptive(at_in, b, tau, spec, rs.RngStream(args.seed))
    torch.cuda.synchronize()
    t_gpu = time.perf_counter() - t0
    g_idx = host(res.row_idx).astype(np.int64)
    g_w = host(res.w)
    g_tr = np.array([[r.k, r.e_schur] for r in res.trace], dtype=np.float64)
    g_resid = rs.row_id_error(a.T, res) / norm_a

    a_host = a.cpu().numpy()
    at = a_host.T
    cores = os.cpu_count() or 1
    with threadpool_limits(limits=cores):
        t0 = time.perf_counter()
        ref = orc.rand_lupp_adaptive(at, b, tau, args.seed, 0, want_w=True)
        t_cpu = time.perf_counter() - t0
    r_idx = np.asarray(ref["row_idx"], dtype=np.int64)
    r_tr = np.array(ref["trace"], dtype=np.float64)
    at_dev = a.T
    w_ref_dev = torch.from_numpy(np.ascontiguousarray(ref["w"])).to(dev)
    r_resid = float(torch.linalg.norm(at_dev - w_ref_dev @ at_dev[torch.from_numpy(r_idx).to(dev)])) / norm_a
    del w_ref_dev

    nt = min(len(g_tr), len(r_tr))
    same_k = bool(nt == 0 or np.array_equal(g_tr[:nt, 0], r_tr[:nt, 0]))
    dtrace = float(np.abs(g_tr[:nt, 1] - r_tr[:nt, 1]).max() / norm_a) if nt else 0.0
    rel_dtrace = float((np.abs(g_tr[:nt, 1] - r_tr[:nt, 1]) / r_tr[:nt, 1]).max()) if nt else 0.0
    w_relerr = None
    if g_w.shape == ref["w"].shape:
        w_relerr = float(np.linalg.norm(g_w - ref["w"]) / np.linalg.norm(ref["w"]))
    tail = lambda tr: [[int(k), float(e), float(e / tau)] for k, e in tr[-4:]]
    out = {
        "layout": "row-major A.T copy" if args.rowmajor else "column-major A.T view",
        "workload": f"cfg2 rand_lupp_adaptive(A.T, b={b}, tau={tau:g} abs) on the {n}x{n} fp64 "
                    f"fast-decay matrix of bench.py (beta=1e-16, Haar bases, seed {args.seed})",
        "norm_a": norm_a,
        "gpu": {"rank": int(res.rank), "status": res.status, "blocks": len(g_tr),
                "seconds_incl_first_call": t_gpu, "resid_rel": g_resid, "trace_tail_k_e_e_over_tau": tail(g_tr)},
        "oracle": {"rank": int(ref["rank"]), "status": ref["status"], "blocks": len(r_tr),
                   "seconds": t_cpu, "cores": cores, "resid_rel": r_resid,
                   "trace_tail_k_e_e_over_tau": tail(r_tr)},
        "rank_equal": int(res.rank) == int(ref["rank"]),
        "status_equal": res.status == ref["status"],
        "row_idx_common_prefix": prefix(g_idx, r_idx),
        "row_idx_set_overlap": len(set(g_idx.tolist()) & set(r_idx.tolist())),
        "trace_k_equal_on_common_blocks": same_k,
        "trace_max_abs_diff_over_norm_a": dtrace,
        "trace_max_rel_diff": rel_dtrace,
        "w_relerr_fro": w_relerr,
    }
    line = json.dumps(out)
    print(line, flush=True)
    if args.out:
        with open(args.out, "w") as f:
            f.write(line + "\n")


if __name__ == "__main__":
    main()
