"""Time the sparse-sign SpMM (`rs_sparse_sign_apply`) against the dense device
form through the DMMA sketch GEMM and the tensor-core (Ozaki) engine, at
m x n x ell (default 20000 x 20000 x 64, zeta 8), with CUDA events."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import paper_2310_09417_b200 as rs  # noqa: E402
from paper_2310_09417_b200 import _device, _lib, _ozaki  # noqa: E402

if os.environ.get("RSKEL_LIB"):  # an experiment build (tools/build_cu_variants.sh)
    _lib.load(os.environ["RSKEL_LIB"])


def timeit(fn, reps=10):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def main():
    m, n, ell, zeta = (int(x) for x in (sys.argv[1:5] if len(sys.argv) > 4 else (20000, 20000, 64, 8)))
    a = torch.randn(m, n, dtype=torch.float64, device="cuda")
    A = _device.as_matrix(a)
    op = rs.make_sketch(rs.SketchSpec("sparsesign", n, ell, zeta=zeta), rs.RngStream(1))
    idx = torch.as_tensor(np.asarray(op.idx, dtype=np.int64)).cuda()
    sg = torch.as_tensor(np.asarray(op.signs)).cuda()
    y = torch.empty(m, ell, dtype=torch.float64, device="cuda")
    plan = torch.empty(int(_lib.load().rs_sparse_sign_plan_bytes(n, ell)), dtype=torch.uint8, device="cuda")
    bad = torch.zeros(1, dtype=torch.int32, device="cuda")

    def spmm():
        _lib.call("rs_sparse_sign_apply", m, n, ell, zeta, A.ptr, A.ld, 0, idx.data_ptr(), sg.data_ptr(),
                  float(op.scale), y.data_ptr(), ell, plan.data_ptr(), bad.data_ptr(), _device.stream_handle())

    om = op.device_dense()
    t_sp = timeit(spmm)
    t_dm = timeit(lambda: _device.sketch_dev(A, om))
    ap = _ozaki.Planes.of_matrix(A)
    bp = _ozaki.Planes(ell, n, _ozaki.OMEGA_PLANES, 64, a.device)
    yo = torch.empty(m, ell, dtype=torch.float64, device="cuda")

    def oz():
        _ozaki.Planes.of_omega(om, out=bp)
        _ozaki.sketch(ap, bp, yo.data_ptr(), ell)

    t_oz = timeit(oz)
    assert int(bad.item()) == 0
    ref = _device.sketch_dev(A, om)
    err = float((y - ref).abs().max() / ref.abs().max())
    gbs = 8.0 * m * n / (t_sp * 1e-3) / 1e9
    print(f"{os.path.basename(os.environ.get('RSKEL_LIB', 'librskel.so'))} m={m} n={n} ell={ell} zeta={zeta}: spmm {t_sp:.3f} ms ({gbs:.0f} GB/s of A), "
          f"dense DMMA {t_dm:.3f} ms, dense tensor-core {t_oz:.3f} ms; max rel diff vs DMMA {err:.1e}")


if __name__ == "__main__":
    main()
