"""cfg3 at full size (32768 x 16384 fp32, tau = 1e-5 ||A||_F): the CUDA adaptive CUR vs the oracle
(the reference composition rand_lupp_adaptive -> _column_skeletons_from_rows -> skeleton.py:639-646,
numpy/OpenBLAS on the host cores) on the same device-generated matrix.  Test infrastructure.

  python tools/cfg3_full_parity.py > profiles/r02_cfg3_full_parity.json
"""
import json
import os
import sys
import time

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
sys.path.insert(0, os.path.join(REPO, "oracle"))


def main():
    import torch
    from threadpoolctl import threadpool_limits

    import paper_2310_09417_b200 as rs
    import randskel_oracle as orc

    m, n, b = 32768, 16384, 64
    a32 = rs.gen_nonneg_lowrank(m, n, 200, 1e-6, rs.RngStream(0).child(1 << 41))
    h32 = a32.cpu().numpy()
    a = h32.astype(np.float64)
    na = float(np.linalg.norm(a))
    tau = 1e-5 * na
    spec = rs.SketchSpec("gaussian", n, b)
    cur, res = rs.cur_decompose_adaptive(a32, b, tau, spec, rs.RngStream(0))
    g_row, g_col = np.asarray(res.row_idx.cpu()), np.asarray(cur.col_idx.cpu())
    u = cur.u_mid.cpu().numpy()
    with threadpool_limits(limits=os.cpu_count()):
        t0 = time.perf_counter()
        ref = orc.rand_lupp_adaptive(a, b, tau, 0, want_w=False)
        r_cur = orc.cur_from_rows(a, ref["row_idx"], ref["rank"])
        cpu_s = time.perf_counter() - t0
    r_row = np.asarray(ref["row_idx"])
    r_col = np.asarray(r_cur["col_idx"])
    u0 = np.asarray(r_cur["u_mid"])

    def resid(rows, cols, um):
        return float(np.linalg.norm(a - a[:, cols] @ (um @ a[rows])) / na)

    out = {"config": "cfg3 32768x16384 fp32 adaptive CUR, tau=1e-5||A||_F", "rank": [res.rank, ref["rank"]],
           "status": [res.status, ref["status"]], "row_idx_equal": bool(np.array_equal(g_row, r_row)),
           "col_idx_equal": bool(np.array_equal(g_col, r_col)),
           "u_mid_rel_diff": float(np.linalg.norm(u - u0) / np.linalg.norm(u0)) if u.shape == u0.shape else None,
           "residual": [resid(g_row, g_col, u), resid(r_row, r_col, u0)], "tau_rel": 1e-5, "cpu_s": cpu_s,
           "cpu_cores": os.cpu_count()}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
