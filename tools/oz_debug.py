"""Exact-integer probe of the tcgen05 kind::i8 path (one plane, one tile)."""
import os
import sys

import numpy as np
import torch

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
sys.path.insert(0, os.path.join(REPO, "tools"))
from oz_check import slice_op  # noqa: E402
from paper_2310_09417_b200 import _device, _lib  # noqa: E402


def run(M, N, K, kmask=None, seed=0):
    g = np.random.default_rng(seed)
    ai = g.integers(-127, 128, size=(M, K))
    bi = g.integers(-127, 128, size=(K, N))
    ai[:, 0] = 127
    bi[0, :] = 127
    if kmask is not None:
        ai[:, kmask:] = 0
        bi[kmask:, :] = 0
        ai[:, 0] = 127
    A = torch.from_numpy(ai / 128.0).cuda()
    B = torch.from_numpy(bi / 128.0).cuda()
    ad, ae, kc = slice_op(A, False, M, K, 1, 128)
    bd, be, _ = slice_op(B, True, N, K, 1, 64)
    Y = torch.zeros(M, N, dtype=torch.float64, device="cuda")
    _lib.call("rs_oz_gemm", M, N, K, kc, 0, 1.0, ad.data_ptr(), ae.data_ptr(), 1, bd.data_ptr(), be.data_ptr(), 1,
              0.0, None, 0, Y.data_ptr(), N, _device.workspace().data_ptr(), _device.stream_handle())
    torch.cuda.synchronize()
    y = np.rint(Y.cpu().numpy() * 128 * 128).astype(np.int64)
    ref = ai @ bi
    np.savez(os.path.join(REPO, "gpurun_out", f"ozdbg_{M}_{N}_{K}_{kmask}.npz"), y=y, ai=ai, bi=bi,
             ad=ad.cpu().numpy(), bd=bd.cpu().numpy())
    bad = y != ref
    print(f"M={M} N={N} K={K} kmask={kmask}: exponents a {np.unique(ae.cpu().numpy())} b {np.unique(be.cpu().numpy())}; "
          f"wrong {bad.sum()} of {bad.size}; rows wrong {np.unique(np.nonzero(bad)[0])[:20]} cols wrong "
          f"{np.unique(np.nonzero(bad)[1])[:20]}", flush=True)
    if bad.any():
        # which k-permutation explains row 0?
        i, j = np.argwhere(bad)[0]
        print("  sample", i, j, y[i, j], ref[i, j])
        # digits of A tile row 0 as stored
        d = ad.cpu().numpy()[:128 * 128].reshape(128, 128)
        print("  stored row0 first 32 bytes", d[0, :32], " expected", ai[0, :32])
    return bad.sum()


if __name__ == "__main__":
    run(128, 64, 128, kmask=32)
    run(128, 64, 128, kmask=64)
    run(128, 64, 128)
    run(128, 64, 256)
    run(256, 128, 512)
