"""Summation-order contract of the DMMA GEMM (include/rskel.h, rs_dgemm) and
the large-panel path.

An output row of a sketch / Schur GEMM must depend only on its row of A, on
B and on K -- not on how many rows are multiplied with it, on the layout of
A, or on whether K arrives in one call or in chunk-aligned pieces.  This is
what makes the column-sharded loop (rows split over ranks) and the host-input
pre-sketch (A multiplied chunk by chunk as it lands) bitwise equal to the
single-GPU device-input path.  Everything here is compared with ``==`` on the
raw bits.
"""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

import randskel_oracle as orc  # noqa: E402


@pytest.fixture(scope="module")
def lib():
    from paper_2310_09417_b200 import _lib

    return _lib


def _ctx():
    from paper_2310_09417_b200 import _device

    return _device.workspace().data_ptr(), _device.stream_handle()


def _gemm(lib, M, N, K, A, lda, colmajor, B, ldb, C, ldc, kc=0, mode=0, Cin=None, ldcin=0, off_a=0, off_c=0):
    ws, st = _ctx()
    lib.call("rs_dgemm_ex", M, N, K, kc, mode, 1.0, A.data_ptr() + 8 * off_a, lda, int(colmajor), None,
             B.data_ptr(), ldb, None, 0.0, Cin.data_ptr() + 8 * off_c if Cin is not None else None, ldcin,
             None, C.data_ptr() + 8 * off_c, ldc, ws, st)


@pytest.mark.parametrize("K", [300, 2500, 20000])
def test_rows_do_not_depend_on_M_or_layout(lib, K):
    """Y = A Omega for all M rows vs for row slices of every size, and for the
    column-major (a.T of a C-ordered matrix) vs the row-major layout."""
    g = torch.Generator(device="cuda").manual_seed(K)
    M, N = 6000, 64
    at = torch.randn(K, M, dtype=torch.float64, device="cuda", generator=g)  # column-major A (M x K)
    om = torch.randn(K, N, dtype=torch.float64, device="cuda", generator=g)
    y = torch.empty(M, N, dtype=torch.float64, device="cuda")
    _gemm(lib, M, N, K, at, M, True, om, N, y, N)
    # the same rows, multiplied in slices of assorted sizes (tile boundaries move)
    ys = torch.empty_like(y)
    bounds = [0, 1, 129, 777, 3000, 3001, 5871, M]
    for lo, hi in zip(bounds[:-1], bounds[1:]):
        _gemm(lib, hi - lo, N, K, at, M, True, om, N, ys, N, off_a=lo, off_c=lo * N)
    # row-major copy of A
    a_row = at.t().contiguous()
    yr = torch.empty_like(y)
    _gemm(lib, M, N, K, a_row, K, False, om, N, yr, N)
    torch.cuda.synchronize()
    ref = torch.from_numpy(np.asarray(at.cpu().numpy().T @ om.cpu().numpy()))
    assert torch.equal(ys, y)
    assert torch.equal(yr, y)
    assert (y.cpu() - ref).abs().max() <= 1e-11 * ref.abs().max()


@pytest.mark.parametrize("K", [400, 20000])
def test_k_pieces_equal_one_shot(lib, K):
    """C = A B fed in chunk-aligned K pieces (RS_GEMM_FOLD across chunks,
    RS_GEMM_CHAIN inside a single chunk) gives the one-shot bits."""
    g = torch.Generator(device="cuda").manual_seed(7)
    M, N = 3000, 128
    at = torch.randn(K, M, dtype=torch.float64, device="cuda", generator=g)
    om = torch.randn(K, N, dtype=torch.float64, device="cuda", generator=g)
    y = torch.empty(M, N, dtype=torch.float64, device="cuda")
    _gemm(lib, M, N, K, at, M, True, om, N, y, N)
    kc = lib.load().rs_gemm_chunk(K)
    if kc < K:
        step, mode, kpass = kc * 3, 1, kc
    else:
        step, mode, kpass = 64, 2, K
    yp = torch.empty_like(y)
    for k0 in range(0, K, step):
        k1 = min(K, k0 + step)
        ws, st = _ctx()
        lib.call("rs_dgemm_ex", M, N, k1 - k0, kpass, 0 if k0 == 0 else mode, 1.0, at.data_ptr() + 8 * k0 * M, M, 1,
                 None, om.data_ptr() + 8 * k0 * N, N, None, 0.0, yp.data_ptr() if k0 else None, N, None,
                 yp.data_ptr(), N, ws, st)
    torch.cuda.synchronize()
    assert torch.equal(yp, y)


def test_sketch_bits_shared_by_pinned_pageable_and_device_input():
    """rand_lupp_adaptive's host-input pre-sketch (row chunks of a pageable or
    pinned array multiplied as they land) and the device-input path produce
    the same trace bits and pivots."""
    import paper_2310_09417_b200 as rs

    n = 3000  # 72 MB: above the pre-sketch threshold
    a, _ = orc.gen_fast_decay(n, n, 1e-16, 0)
    at = np.ascontiguousarray(a)  # column ID of `a`: the candidates are columns
    tau = 1e-9 * np.linalg.norm(a)
    spec = rs.SketchSpec("gaussian", n, 64)
    dev = rs.rand_lupp_adaptive(torch.from_numpy(at).cuda().T, 64, tau, spec, rs.RngStream(0))
    page = rs.rand_lupp_adaptive(at.T, 64, tau, spec, rs.RngStream(0))
    pinned = torch.from_numpy(at).pin_memory().numpy()
    pin = rs.rand_lupp_adaptive(pinned.T, 64, tau, spec, rs.RngStream(0))
    tr = lambda r: np.array([x.e_schur for x in r.trace])  # noqa: E731
    for r in (page, pin):
        assert r.rank == dev.rank
        assert np.array_equal(np.asarray(r.row_idx), dev.row_idx.cpu().numpy())
        assert np.array_equal(tr(r), tr(dev))


def test_panel_beyond_shared_memory(lib):
    """R = 100,000 candidate rows (more than 148 x 227 KB of shared memory
    holds): rows stay in global memory, pivots and factors are the
    unblocked panel's (numpy rounding), bit for bit."""
    R, w = 100000, 64
    a = np.random.default_rng(11).standard_normal((R, w))
    S = torch.from_numpy(a.copy()).cuda()
    perm = torch.empty(R, dtype=torch.int64, device="cuda")
    nc = torch.zeros(1, dtype=torch.int32, device="cuda")
    ws, st = _ctx()
    lib.call("rs_panel_lupp", S.data_ptr(), w, R, w, perm.data_ptr(), nc.data_ptr(), ws, st)
    torch.cuda.synchronize()
    L0, U0, perm0, nc0 = orc.lupp(a)
    assert int(nc.item()) == 64 == nc0
    p = perm.cpu().numpy()
    assert np.array_equal(p, perm0)
    s = S.cpu().numpy()[p]
    assert np.array_equal(np.triu(s[:w]), U0)
    assert np.array_equal(np.tril(s, -1)[:, :w] + np.eye(R, w), L0)
