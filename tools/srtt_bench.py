"""SRTT embedding: the FFT form (`rs_srtt_apply`) vs the dense embedding through the DMMA
sketch GEMM and the tensor-core engine, m x n x ell (CUDA events).
python tools/srtt_bench.py [m n ell ...]"""
import os
import sys

import torch

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import paper_2310_09417_b200 as rs  # noqa: E402
from paper_2310_09417_b200 import _device, _ozaki  # noqa: E402


def timeit(fn, reps=5):
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
    args = [int(x) for x in sys.argv[1:]] or [20000, 20000, 64, 20000, 20000, 256, 20000, 20000, 1024]
    for m, n, ell in zip(args[0::3], args[1::3], args[2::3]):
        a = torch.randn(m, n, dtype=torch.float64, device="cuda")
        A = _device.as_matrix(a)
        op = rs.make_sketch(rs.SketchSpec("srtt", n, ell), rs.RngStream(1))
        t_fft = timeit(lambda: _device.srtt_apply(A, op.perm, op.signs, op.cols, op.scale))
        om = op.device_dense()
        t_dm = timeit(lambda: _device.sketch_dev(A, om))
        ap = _ozaki.Planes.of_matrix(A)
        bp = _ozaki.Planes(ell, n, _ozaki.OMEGA_PLANES, 64, a.device)
        yo = torch.empty(m, ell, dtype=torch.float64, device="cuda")

        def oz():
            _ozaki.Planes.of_omega(om, out=bp)
            _ozaki.sketch(ap, bp, yo.data_ptr(), ell)

        t_oz = timeit(oz)
        t_om = timeit(lambda: op.device_dense())
        print(f"m={m} n={n} ell={ell}: fft {t_fft:.3f} ms | dense DMMA {t_dm:.3f} ms | dense tensor-core "
              f"{t_oz:.3f} ms (+ dense Omega {t_om:.3f} ms)", flush=True)
        del ap, bp, a, A


if __name__ == "__main__":
    main()
