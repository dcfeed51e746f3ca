"""cfg3 (BASELINE configs[2]): adaptive CUR of a 32768 x 16384 fp32 non-negative low-rank-plus-noise
matrix, tau = 1e-5 ||A||_F.  Per-stage CUDA-event times, both sketch engines.
   python tools/cfg3_profile.py"""
import json
import os
import sys

import torch

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
import paper_2310_09417_b200 as rs  # noqa: E402
from paper_2310_09417_b200 import _device, _ozaki, cur, skeleton  # noqa: E402

m, n, r0, b = 32768, 16384, 200, 64
a32 = rs.gen_nonneg_lowrank(m, n, r0, 1e-6, rs.RngStream(0).child(1 << 41))
tau = 1e-5 * float(torch.linalg.norm(a32.double()))
spec = rs.SketchSpec("gaussian", n, b)


def ev():
    e = torch.cuda.Event(enable_timing=True)
    e.record()
    return e


for engine in ("ozaki", "dmma"):
    rs.set_sketch_engine(engine)
    for rep in range(3):
        torch.cuda.synchronize()
        t = [ev()]
        A = _device.as_matrix(a32)
        planes = _ozaki.Planes.of_matrix(A) if engine == "ozaki" else None
        t.append(ev())
        res = skeleton._adaptive_device(A, b, tau, spec, rs.RngStream(0), planes=planes)
        t.append(ev())
        ridx = cur._idx(res.row_idx)
        k = res.rank
        cidx, _ = cur._column_skeletons_from_rows(A, ridx, k)
        C = cur._cols(A, cidx)
        R = cur._rows(A, ridx)
        t.append(ev())
        arp_t = cur._pinv_apply_dev(R.T, A.T, b_planes=planes)
        t.append(ev())
        u_mid = cur._pinv_apply_dev(C, cur.dense._mat(arp_t).T)
        t.append(ev())
        c1 = cur._cond1(cur._cols(R, cidx))
        t.append(ev())
        torch.cuda.synchronize()
        whole0 = ev()
        cf, rr = rs.cur_decompose_adaptive(a32, b, tau, spec, rs.RngStream(0))
        whole1 = ev()
        torch.cuda.synchronize()
        names = ["upcast+planes", "adaptive ID (rows)", "column skeletons+gathers", "pinv(R^T, A^T)", "pinv(C, .)",
                 "cond1"]
        out = {"engine": engine, "rep": rep, "rank": k, "status": res.status, "cur_status": cf.status,
               "whole_ms": whole0.elapsed_time(whole1)}
        out.update({nm: round(t[i].elapsed_time(t[i + 1]), 3) for i, nm in enumerate(names)})
        print(json.dumps(out), flush=True)
rs.set_sketch_engine("ozaki")
