"""CUDA path vs the reference (golden fixtures) and the CPU oracle.

Parity bar: skeleton indices / pivot order identical; rank
and status identical; e_schur trace within 1e-12 * ||A||_F absolute;
interpolation matrices within 1e-10 relative (fp64 GEMM/solve rounding
differs from OpenBLAS/LAPACK, indices may not).
"""

import ctypes
import os
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

import randskel_oracle as orc  # noqa: E402
from conftest import golden  # noqa: E402


@pytest.fixture(scope="module")
def rs():
    import paper_2310_09417_b200 as rs

    return rs


def spec(rs, n, ell=None):
    return rs.SketchSpec("gaussian", n=n, ell=ell or min(n, 32))


def relerr(x, y):
    x = np.asarray(x)
    y = np.asarray(y)
    return np.linalg.norm(x - y) / max(np.linalg.norm(y), 1e-300)


# Residual tolerance (fp64): the interpolation matrix of a numerically
# rank-deficient sketch is ill-conditioned, so entrywise W differences between
# two fp64 implementations scale with cond(L1) * eps.  The quantity the ID
# certifies -- the relative residual ||A - W A[I]|| / ||A|| -- must agree to
# within 50% of the reference's value plus 1e-13 (pure rounding floor).
RESID_REL, RESID_ABS = 0.5, 1e-13


def assert_resid_close(ours, ref):
    assert ours <= (1 + RESID_REL) * ref + RESID_ABS, (ours, ref)
    assert ref <= (1 + RESID_REL) * ours + RESID_ABS, (ours, ref)


def row_resid(a, idx, w):
    return np.linalg.norm(a - w @ a[idx]) / np.linalg.norm(a)


def col_resid(a, idx, x):
    return np.linalg.norm(a - a[:, idx] @ x) / np.linalg.norm(a)


def common_prefix(a, b):
    n = min(len(a), len(b))
    d = np.nonzero(np.asarray(a[:n]) != np.asarray(b[:n]))[0]
    return n if d.size == 0 else int(d[0])


# ----------------------------------------------------------------- GEMM ----
@pytest.mark.parametrize("M,N,K", [(1, 1, 1), (7, 5, 3), (128, 64, 16), (300, 70, 129),
                                    (513, 257, 1000), (64, 1, 0)])
@pytest.mark.parametrize("colmajor", [False, True])
def test_dgemm_matches_fp64(rs, M, N, K, colmajor):
    from paper_2310_09417_b200 import _device

    g = np.random.default_rng(M * 7 + N * 3 + K)
    a = g.standard_normal((M, K))
    b = g.standard_normal((K, N))
    c = g.standard_normal((M, N))
    A = _device.as_matrix(np.asfortranarray(a) if colmajor else a)
    assert A.colmajor == (colmajor and M > 1 and K > 1)
    B = _device.as_matrix(b)
    C = _device.as_matrix(c)
    out = _device.dgemm(A, B, alpha=-1.0, beta=1.0, cin=C).cpu().numpy()
    ref = c - a @ b
    scale = max(1.0, np.abs(a).sum(1).max(initial=0.0) * np.abs(b).max(initial=0.0))
    assert np.abs(out - ref).max(initial=0.0) <= 1e-13 * scale


def test_dgemm_row_gathers(rs):
    from paper_2310_09417_b200 import _device

    g = np.random.default_rng(3)
    a = g.standard_normal((90, 33))
    b = g.standard_normal((50, 17))
    c = g.standard_normal((70, 17))
    ai = g.permutation(90)[:40]
    bi = g.permutation(50)[:33]
    ci = g.permutation(70)[:40]
    out = _device.dgemm(
        _device.as_matrix(a), _device.as_matrix(b), alpha=2.0, beta=-0.5, cin=_device.as_matrix(c),
        aidx=_device.as_index(ai, "numpy"), bidx=_device.as_index(bi, "numpy"),
        cidx=_device.as_index(ci, "numpy"),
    )
    ref = 2.0 * a[ai] @ b[bi] - 0.5 * c[ci]
    assert np.abs(out.cpu().numpy() - ref).max() <= 1e-12


# ---------------------------------------------------------------- panel ----
def _panel(rs, s):
    from paper_2310_09417_b200 import _device, _lib

    s = np.ascontiguousarray(s, dtype=np.float64)
    R, w = s.shape
    S = torch.as_tensor(s).cuda()
    perm = torch.empty(R, dtype=torch.int64, device="cuda")
    nc = torch.empty(1, dtype=torch.int32, device="cuda")
    _lib.call("rs_panel_lupp", S.data_ptr(), w, R, w, perm.data_ptr(), nc.data_ptr(),
              _device.workspace().data_ptr(), _device.stream_handle())
    return S.cpu().numpy(), perm.cpu().numpy(), int(nc.item())


def _split(s_fact, perm, nc):
    P = s_fact[perm]
    L = np.tril(P[:, :nc], -1)
    L[np.arange(nc), np.arange(nc)] = 1.0
    U = np.triu(P[:nc, :nc])
    return L, U


@pytest.mark.parametrize("case", ["lupp_tiebreak", "lupp_hand", "lupp_chan5", "lupp_chan10",
                                  "lupp_chan20", "lupp_chan30"])
def test_panel_known_answers(rs, case):
    g = golden(case)
    n = g["U"].shape[0]
    if case == "lupp_tiebreak":
        a = np.array([[1, 5], [1, 5], [3, 0], [1, 1]], dtype=float)
    elif case == "lupp_hand":
        a = np.array([[1, 2], [3, 4]], dtype=float)
    else:
        a = orc.gen_chan(n)
    s, perm, nc = _panel(rs, a)
    assert nc == a.shape[1]
    assert np.array_equal(perm, g["perm"])
    L, U = _split(s, perm, nc)
    # numpy rounding is reproduced exactly inside a panel (mul, then sub)
    assert np.array_equal(L, g["L"]) and np.array_equal(U, g["U"])
    if case.startswith("lupp_chan"):
        assert np.abs(U).max() / np.abs(a).max() == 2.0 ** (n - 1)


@pytest.mark.parametrize("seed", [0, 1])
def test_panel_random_matches_reference(rs, seed):
    g = golden(f"lupp_rand{seed}")
    m, k = int(g["m"]), int(g["k"])
    a = np.random.default_rng(seed).standard_normal((m, k))
    s, perm, nc = _panel(rs, a)
    assert nc == k and np.array_equal(perm, g["perm"])
    L, U = _split(s, perm, nc)
    assert np.abs(L - g["L"]).max() <= 1e-13 and np.abs(U - g["U"]).max() <= 1e-13


def test_panel_zero_pivot_partial(rs):
    col0 = np.array([4.0, 2.0, 8.0, 1.0])
    col1 = np.array([1.0, 2.0, 4.0, 8.0])
    a = np.column_stack([col0, col1, col0])
    _, _, nc = _panel(rs, a)
    assert nc == 2


def test_panel_large_multi_cta(rs):
    """Rows spread over all SMs: compare with the oracle's unblocked panel."""
    a = np.random.default_rng(9).standard_normal((20000, 64))
    s, perm, nc = _panel(rs, a)
    L0, U0, perm0, nc0 = orc.lupp(a)
    assert nc == 64 and np.array_equal(perm, perm0)
    L, U = _split(s, perm, nc)
    assert relerr(U, U0) < 1e-13


# ------------------------------------------------------ fixed-rank IDs ----
def test_rand_lupp_exact_rank(rs):
    g = golden("rand_lupp_exact")
    r = rs.rand_lupp(g["a"], 30, spec(rs, 80), rs.RngStream(1))
    assert np.array_equal(r.row_idx, g["row_idx"])
    assert relerr(r.w, g["w"]) < 1e-10
    assert np.array_equal(r.w[r.row_idx], np.eye(30))


@pytest.mark.parametrize("k", [40, 150])
def test_rand_lupp_and_column_id_fast_decay(rs, k):
    a = golden("fast_decay_300")["a"]
    g = golden(f"rand_lupp_fd300_k{k}")
    r = rs.rand_lupp(a, k, spec(rs, 300), rs.RngStream(int(g["seed"])))
    assert np.array_equal(r.row_idx, g["row_idx"])
    assert_resid_close(row_resid(a, r.row_idx, r.w), float(g["resid"]))
    if k <= 40:  # well-conditioned L1: entrywise agreement too
        assert relerr(r.w, g["w"]) < 1e-10
    g = golden(f"column_id_fd300_k{k}")
    c = rs.column_id(a, k, spec(rs, 300), rs.RngStream(int(g["seed"])))
    assert np.array_equal(c.col_idx, g["col_idx"])
    assert_resid_close(col_resid(a, c.col_idx, c.x), float(g["resid"]))
    if k <= 40:
        assert relerr(c.x, g["x"]) < 1e-10
    assert np.array_equal(c.x[:, c.col_idx], np.eye(k))


def test_column_id_k256(rs):
    g = golden("column_id_fd1000_k256")
    a, _ = orc.gen_fast_decay(1000, 1000, 1e-16, int(g["gen_seed"]))
    assert abs(a.sum() - float(g["a_sum"])) < 1e-10
    c = rs.column_id(a, 256, rs.SketchSpec("gaussian", 1000, 256), rs.RngStream(0))
    assert np.array_equal(c.col_idx, g["col_idx"])
    assert_resid_close(col_resid(a, c.col_idx, c.x), float(g["resid"]))
    assert relerr(c.x[:, :16], g["x_head"]) < 1e-9


def test_rank_deficient_raises(rs):
    with pytest.raises(rs.RankDeficientError):
        rs.rand_lupp(np.zeros((20, 10)), 5, spec(rs, 10), rs.RngStream(4))


# ---------------------------------------------------------- adaptive ID ----
ADAPTIVE_CASES = ["adapt_fd200", "adapt_fd150_s0", "adapt_fd150_s1", "adapt_fd150_s2",
                  "adapt_notconv", "adapt_exhausted", "adapt_wide", "adapt_b25",
                  "adapt_fullwidth", "adapt_single", "adapt_maxrank0", "adapt_maxrank15"]


@pytest.mark.parametrize("case", ADAPTIVE_CASES)
def test_adaptive_matches_reference(rs, case):
    g = golden(case)
    a = g["a"]
    mr = int(g["max_rank"])
    res = rs.rand_lupp_adaptive(a, int(g["b"]), float(g["tau"]), spec(rs, a.shape[1], int(g["b"])),
                                rs.RngStream(int(g["seed"])), max_rank=None if mr < 0 else mr)
    assert res.status == str(g["status"])
    assert res.rank == int(g["rank"])
    na = np.linalg.norm(a)
    if float(g["tau"]) >= 1e-12 * na:
        assert np.array_equal(res.row_idx, g["row_idx"])
    else:
        # tau at the fp64 noise floor: the last pivots are chosen among
        # rounding-level Schur entries and are not well separated.
        assert common_prefix(res.row_idx, g["row_idx"]) >= res.rank - int(g["b"])
        assert len(set(res.row_idx.tolist()) & set(g["row_idx"].tolist())) >= res.rank - 2
    tr = np.array([[r.k, r.e_schur] for r in res.trace])
    assert np.array_equal(tr[:, 0], g["trace"][:, 0])
    assert np.abs(tr[:, 1] - g["trace"][:, 1]).max() <= 1e-12 * na
    assert_resid_close(row_resid(a, res.row_idx, res.w), float(g["resid"]))
    assert np.array_equal(res.w[res.row_idx], np.eye(res.rank))


@pytest.mark.parametrize("tau_rel", ["1e-08", "0.0001"])
def test_adaptive_criterion4_ranks(rs, tau_rel):
    g = golden(f"adapt_crit4_{tau_rel}")
    a, _ = orc.gen_fast_decay(1000, 1000, 1e-16, int(g["gen_seed"]))
    res = rs.rand_lupp_adaptive(a, 50, float(g["tau"]), spec(rs, 1000, 50), rs.RngStream(0))
    assert res.rank == int(g["rank"]) and res.status == "ok"
    assert np.array_equal(res.row_idx, g["row_idx"])
    tr = np.array([r.e_schur for r in res.trace])
    assert np.abs(tr - g["trace"][:, 1]).max() <= 1e-12 * np.linalg.norm(a)


def test_adaptive_cfg2_shape_n2000(rs):
    """cfg2 recipe (column ID via a.T, b = 64, absolute tau = 1e-8) at n = 2000."""
    g = golden("adapt_cfg2_n2000")
    a, _ = orc.gen_fast_decay(2000, 2000, 1e-16, 0, orc.child_stream(0, 1 << 41))
    assert abs(a.sum() - float(g["a_sum"])) < 1e-9
    res = rs.rand_lupp_adaptive(a.T, 64, 1e-8, spec(rs, 2000, 64), rs.RngStream(0))
    assert res.rank == int(g["rank"]) == 1344
    assert res.status == "ok"
    assert np.array_equal(res.row_idx, g["row_idx"])
    tr = np.array([r.e_schur for r in res.trace])
    assert np.abs(tr - g["trace"][:, 1]).max() <= 1e-12 * np.linalg.norm(a)
    assert_resid_close(row_resid(a.T, res.row_idx, res.w), float(g["resid"]))


def test_adaptive_device_tensor_roundtrip(rs):
    """CUDA tensor in -> CUDA tensors out, same answer as the numpy path."""
    g = golden("adapt_fd200")
    a = g["a"]
    res = rs.rand_lupp_adaptive(torch.as_tensor(a).cuda(), 20, float(g["tau"]), spec(rs, 200, 20),
                                rs.RngStream(25))
    assert res.w.is_cuda and res.row_idx.is_cuda
    assert np.array_equal(res.row_idx.cpu().numpy(), g["row_idx"])


def test_adaptive_argument_errors(rs):
    a = np.eye(10)
    with pytest.raises(ValueError):
        rs.rand_lupp_adaptive(a, 2, 0.0, spec(rs, 10), rs.RngStream(0))
    with pytest.raises(rs.DimensionError):
        rs.rand_lupp_adaptive(a, 11, 1.0, spec(rs, 10), rs.RngStream(0))


def test_adaptive_nonfinite_rejected(rs):
    a = np.ones((40, 30))
    a[3, 4] = np.nan
    with pytest.raises(ValueError):
        rs.rand_lupp_adaptive(a, 8, 1e-3, spec(rs, 30), rs.RngStream(0))


@pytest.mark.parametrize("b", [64, 32])
def test_adaptive_rank_exhausted_full_width_block(b):
    """Zero pivot in the middle of a b-wide block on the speculative
    (absorb-ahead) path: the block is re-absorbed truncated from its own
    factored Schur block (`skeleton.py:439-454`, `dense.py:195-198`)."""
    import paper_2310_09417_b200 as rs

    g = np.random.default_rng(41)
    a = np.zeros((500, 400))
    rows = np.sort(g.choice(500, 100, replace=False))
    a[rows] = g.standard_normal((100, 400))
    spec = rs.SketchSpec("gaussian", 400, b)
    res = rs.rand_lupp_adaptive(a, b, 1e-30, spec, rs.RngStream(3))
    ref = orc.rand_lupp_adaptive(a, b, 1e-30, 3)
    assert res.status == ref["status"] == "rank_exhausted"
    assert res.rank == ref["rank"] == 100
    assert np.array_equal(np.sort(res.row_idx), rows)
    assert np.array_equal(res.row_idx, ref["row_idx"])
    err = np.linalg.norm(a - res.w @ a[res.row_idx]) / np.linalg.norm(a)
    assert err <= 1e-12


@pytest.mark.parametrize("ld_pad", [0, 1])
def test_gather_kernels_match_numpy(rs, ld_pad):
    """rs_gather_rows / rs_gather2d against numpy fancy indexing, for the vectorised path
    (even leading dimensions) and the scalar path (odd), narrow and wide rows, both source
    layouts, and idx < 0 = zero row (`skeleton.py:569,619,639-645`)."""
    import torch
    from paper_2310_09417_b200 import _lib, _device

    g = np.random.default_rng(7)
    st = _device.stream_handle()
    for rows, cols in ((300, 64), (257, 5000), (40, 3)):
        ld = cols + ld_pad
        a = g.standard_normal((rows, ld))
        dev = torch.from_numpy(a).cuda()
        idx = g.integers(0, rows, size=rows + 17)
        idx[5] = -1
        out = torch.full((idx.size, cols), np.nan, dtype=torch.float64, device="cuda")
        idx_d = torch.from_numpy(idx).cuda()
        _lib.call("rs_gather_rows", dev.data_ptr(), ld, idx_d.data_ptr(), idx.size, cols, out.data_ptr(), cols, st)
        ref = a[np.maximum(idx, 0), :cols].copy()
        ref[5] = 0.0
        assert np.array_equal(out.cpu().numpy(), ref)
        # 2-D: rows and columns, row-major and column-major source
        I = g.integers(0, rows, size=min(rows, 33))
        J = g.integers(0, cols, size=min(cols, 70))
        for colmajor in (False, True):
            src = np.asfortranarray(a[:, :cols]) if colmajor else a
            t = torch.from_numpy(src.T.copy() if colmajor else src).cuda()
            rs_, cs_ = (1, rows) if colmajor else (ld, 1)
            for ri, ci in ((I, None), (None, J), (I, J)):
                nr = rows if ri is None else ri.size
                nc = cols if ci is None else ci.size
                o = torch.full((nr, nc), np.nan, dtype=torch.float64, device="cuda")
                rid = torch.from_numpy(ri).cuda() if ri is not None else None  # kept alive for the call
                cid = torch.from_numpy(ci).cuda() if ci is not None else None
                _lib.call("rs_gather2d", t.data_ptr(), rs_, cs_, rid.data_ptr() if rid is not None else None, nr,
                          cid.data_ptr() if cid is not None else None, nc, o.data_ptr(), nc, st)
                want = a[:, :cols][ri if ri is not None else slice(None)]
                want = want[:, ci] if ci is not None else want
                assert np.array_equal(o.cpu().numpy(), want), (rows, cols, colmajor, ri is None, ci is None)
