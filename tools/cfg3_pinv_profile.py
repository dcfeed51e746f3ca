"""Sub-steps of the two compressed min-norm solves of the cfg3 CUR (U = C^+ A R^+), CUDA events
around each (the host waits where the code reads a device flag).  python tools/cfg3_pinv_profile.py"""
import json
import os
import sys

import torch

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
import paper_2310_09417_b200 as rs  # noqa: E402
from paper_2310_09417_b200 import _device, _engine, _lib, _ozaki, cur, dense, skeleton  # noqa: E402

m, n, r0, b = 32768, 16384, 200, 64
a32 = rs.gen_nonneg_lowrank(m, n, r0, 1e-6, rs.RngStream(0).child(1 << 41))
tau = 1e-5 * float(torch.linalg.norm(a32.double()))
spec = rs.SketchSpec("gaussian", n, b)


def ev():
    e = torch.cuda.Event(enable_timing=True)
    e.record()
    return e


def pinv_steps(A, B, b_planes=None):
    p, q = A.shape
    r = B.cols
    dev = _device.device()
    T = [("start", ev())]
    Ar = A.row_major()
    T.append(("row_major", ev()))
    st, W, fail = _engine.factor_sample(Ar, want_w=True)
    T.append(("LUPP + W", ev()))
    Wm = dense._mat(W)
    A_I = cur._rows(Ar, st.perm[:q].clone())
    G = torch.empty((q, q), dtype=torch.float64, device=dev)
    dense._gemm(dense._mat(G), Wm.T, Wm)
    status = torch.empty(1, dtype=torch.int32, device=dev)
    _lib.call("rs_cholesky", G.data_ptr(), q, q, status.data_ptr(), cur._st())
    ok = int(status.item())
    T.append(("W^T W + Cholesky (+ host read)", ev()))
    Rw = dense._mat(G)
    M = torch.empty((q, q), dtype=torch.float64, device=dev)
    dense._gemm(dense._mat(M), Rw, A_I)
    T.append(("M = R_W A[I]", ev()))
    if B.colmajor and b_planes is not None and b_planes.rows == r and b_planes.K == p:
        Ht = torch.empty((r, q), dtype=torch.float64, device=dev)
        om = _ozaki.Planes.of_omega(W)
        T.append(("W digit planes", ev()))
        _ozaki.sketch(b_planes, om, Ht.data_ptr(), q)
        T.append(("H^T = B^T W (tensor cores)", ev()))
        H = dense._mat(Ht).T.row_major()
    elif B.colmajor:
        Ht = torch.empty((r, q), dtype=torch.float64, device=dev)
        dense._gemm(dense._mat(Ht), B.T, Wm)
        T.append(("H^T = B^T W (DMMA)", ev()))
        H = dense._mat(Ht).T.row_major()
    else:
        Hr = torch.empty((q, r), dtype=torch.float64, device=dev)
        dense._gemm(dense._mat(Hr), Wm.T, B)
        H = dense._mat(Hr)
        T.append(("H = W^T B (DMMA)", ev()))
    T.append(("H layout", ev()))
    H2 = dense._trsm_left(Rw.T, H, lower=True, unit=False)
    T.append(("TRSM R_W^T", ev()))
    Mm = dense._mat(M)
    c = cur._cond1(Mm)
    T.append(("cond1(M) (+ host read)", ev()))
    x = cur._lu_solve(Mm, H2) if c < 1e10 else None
    T.append(("LU solve", ev()))
    torch.cuda.synchronize()
    return x, {nm: round(T[i - 1][1].elapsed_time(T[i][1]), 3) for i, (nm, _) in enumerate(T) if i > 0}


for rep in range(3):
    A = _device.as_matrix(a32)
    planes = _ozaki.Planes.of_matrix(A)
    res = skeleton._adaptive_device(A, b, tau, spec, rs.RngStream(0), planes=planes)
    ridx = cur._idx(res.row_idx)
    k = res.rank
    cidx, _ = cur._column_skeletons_from_rows(A, ridx, k)
    C = cur._cols(A, cidx)
    R = cur._rows(A, ridx)
    torch.cuda.synchronize()
    arp_t, s1 = pinv_steps(R.T, A.T, b_planes=planes)
    _, s2 = pinv_steps(C, dense._mat(arp_t).T)
    print(json.dumps({"rep": rep, "k": k, "pinv(R^T, A^T)": s1, "pinv(C, .)": s2}), flush=True)
