"""Where the cfg3 adaptive-CUR time goes (CUDA events per stage).
   PYTHONPATH=. python tools/cfg3_profile.py"""
import time

import torch

import paper_2310_09417_b200 as rs
from paper_2310_09417_b200 import _device, cur, dense

m, n, r0, b = 32768, 16384, 200, 64
g = torch.Generator(device="cuda")
g.manual_seed(0)
w = torch.rand(m, r0, generator=g, dtype=torch.float64, device="cuda")
h = torch.rand(r0, n, generator=g, dtype=torch.float64, device="cuda")
low = w @ h
noise = torch.rand(m, n, generator=g, dtype=torch.float64, device="cuda")
a32 = (low + 1e-6 * torch.linalg.norm(low) / torch.linalg.norm(noise) * noise).to(torch.float32)
del low, noise, w, h
tau = 1e-5 * float(torch.linalg.norm(a32.double()))
spec = rs.SketchSpec("gaussian", n, b)


def ev():
    e = torch.cuda.Event(enable_timing=True)
    e.record()
    return e


for rep in range(2):
    torch.cuda.synchronize()
    t = [ev()]
    A = _device.as_matrix(a32)
    t.append(ev())
    res = rs.rand_lupp_adaptive(A, b, tau, spec, rs.RngStream(0))
    t.append(ev())
    ridx = cur._idx(res.row_idx)
    k = res.rank
    cidx, _ = cur._column_skeletons_from_rows(A, ridx, k)
    t.append(ev())
    C = cur._cols(A, cidx)
    R = cur._rows(A, ridx)
    t.append(ev())
    arp_t = cur._pinv_apply_dev(R.T, A.T)
    t.append(ev())
    u_mid = cur._pinv_apply_dev(C, dense._mat(arp_t).T)
    t.append(ev())
    S = cur._cols(R, cidx)
    c1 = cur._cond1(S)
    t.append(ev())
    torch.cuda.synchronize()
    names = ["upcast", "adaptive ID (rows)", "column skeletons", "gathers", "pinv(R^T, A^T)", "pinv(C, .)", "cond1"]
    print(f"rep {rep}: rank {k}: " + ", ".join(f"{nm} {t[i].elapsed_time(t[i + 1]):.1f} ms"
                                               for i, nm in enumerate(names)))
