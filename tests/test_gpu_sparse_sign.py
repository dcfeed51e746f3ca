"""Sparse-sign embedding applied as an SpMM on the device (`rs_sparse_sign_apply`)
against the reference's `SparseSignSketch.apply` (`sketching.py:176-185`): the
golden outputs and the oracle's csc_matvecs-order restatement, bit for bit."""
import ctypes

import numpy as np
import pytest

from conftest import golden  # noqa: E402

pytestmark = pytest.mark.gpu

import randskel_oracle as orc  # noqa: E402


def _rs():
    import paper_2310_09417_b200 as rs
    return rs


def test_golden_both_sides_bitwise():
    rs = _rs()
    g = golden("sketch_sparsesign")
    a = np.random.default_rng(80).standard_normal((90, 70))
    op = rs.make_sketch(rs.SketchSpec("sparsesign", 70, 16, zeta=4), rs.RngStream(81))
    assert np.array_equal(rs.apply_sketch(a, op), g["y"])
    assert np.array_equal(op.apply(a), g["y"])
    op2 = rs.make_sketch(rs.SketchSpec("sparsesign", 90, 16, zeta=4), rs.RngStream(82))
    assert np.array_equal(rs.apply_sketch(a, op2, side="transposed_right"), g["yt"])


@pytest.mark.parametrize("m,n,ell,zeta,layout", [
    (1, 2, 2, 2, "row"), (3, 31, 5, 2, "row"), (129, 33, 7, 7, "col"), (1000, 2000, 64, 8, "row"),
    (1000, 2000, 64, 8, "col"), (300, 777, 33, 3, "row"), (257, 513, 200, 8, "row"), (200, 300, 130, 130, "col"),
    (64, 4096, 32, 8, "col"),
])
def test_random_shapes_vs_oracle_bitwise(m, n, ell, zeta, layout):
    """Ragged row blocks, partial 32-row chunks, ell <= 32, ell > 64 (column groups),
    zeta = ell, both layouts of A, wide dynamic range in A."""
    import torch

    rs = _rs()
    gen = np.random.default_rng(m * 7 + n)
    a = gen.standard_normal((m, n)) * np.exp(3 * gen.standard_normal((m, n)))
    op = rs.make_sketch(rs.SketchSpec("sparsesign", n, ell, zeta=zeta), rs.RngStream(m + n))
    want = orc.sparse_sign_apply(a, np.asarray(op.idx), np.asarray(op.signs), op.scale, ell)
    src = a if layout == "row" else np.asfortranarray(a)
    got = rs.apply_sketch(torch.as_tensor(src).cuda(), op).cpu().numpy()
    assert np.array_equal(got.view(np.int64), want.view(np.int64))


def test_fp32_input_is_upcast_exactly():
    rs = _rs()
    gen = np.random.default_rng(5)
    a = gen.standard_normal((150, 400)).astype(np.float32)
    op = rs.make_sketch(rs.SketchSpec("sparsesign", 400, 24, zeta=6), rs.RngStream(6))
    want = orc.sparse_sign_apply(a.astype(np.float64), np.asarray(op.idx), np.asarray(op.signs), op.scale, 24)
    assert np.array_equal(rs.apply_sketch(a, op), want)


def test_hand_built_operator_outside_the_spmm_uses_the_dense_form():
    """Signs other than +-1 (the reference accepts any) go through the dense device form."""
    rs = _rs()
    from paper_2310_09417_b200.sketching import SparseSignSketch

    gen = np.random.default_rng(9)
    idx = np.stack([gen.permutation(12)[:3] for _ in range(50)])
    signs = gen.standard_normal((50, 3))
    op = SparseSignSketch(idx, signs, 12, 0.5)
    assert not op.spmm_exact()
    a = gen.standard_normal((20, 50))
    want = orc.sparse_sign_apply(a, idx, signs, 0.5, 12)
    np.testing.assert_allclose(op.apply(a), want, rtol=1e-13, atol=1e-13)


def test_abi_flags_invalid_operators():
    """The C ABI sets `bad`: 1 for an index outside [0, ell) or a sign other than +-1,
    2 for an index repeated within a row."""
    import torch

    from paper_2310_09417_b200 import _device, _lib

    lib = _lib.load()
    dev = torch.device("cuda:0")
    n, ell, zeta, m = 40, 8, 3, 10
    a = torch.randn(m, n, dtype=torch.float64, device=dev)
    y = torch.empty(m, ell, dtype=torch.float64, device=dev)
    plan = torch.empty(int(lib.rs_sparse_sign_plan_bytes(n, ell)), dtype=torch.uint8, device=dev)
    good = np.stack([np.random.default_rng(i).permutation(ell)[:zeta] for i in range(n)])
    for case, want in (("ok", 0), ("range", 1), ("sign", 1), ("repeat", 2)):
        idx = good.copy()
        sg = np.ones((n, zeta))
        if case == "range":
            idx[5, 1] = ell
        elif case == "sign":
            sg[7, 2] = 0.5
        elif case == "repeat":
            idx[3, 1] = idx[3, 0]
        idx_d = torch.as_tensor(idx.astype(np.int64)).to(dev)
        sg_d = torch.as_tensor(sg).to(dev)
        bad = torch.zeros(1, dtype=torch.int32, device=dev)
        st = lib.rs_sparse_sign_apply(m, n, ell, zeta, ctypes.c_void_p(a.data_ptr()), n, 0,
                                      ctypes.c_void_p(idx_d.data_ptr()), ctypes.c_void_p(sg_d.data_ptr()), 0.5,
                                      ctypes.c_void_p(y.data_ptr()), ell, ctypes.c_void_p(plan.data_ptr()),
                                      ctypes.c_void_p(bad.data_ptr()), ctypes.c_void_p(_device.stream_handle()))
        assert st == 0
        assert int(bad.item()) & want == want and (want or int(bad.item()) == 0), case


def test_adaptive_loop_sparse_sign_sketches_are_the_references():
    """The adaptive loop's sparse-sign blocks use the SpMM: Y_t is bitwise the
    reference operator's product, so the loop follows the reference's golden case."""
    rs = _rs()
    ga = golden("adapt_sparsesign")
    gg = np.random.default_rng(84)
    b_exact = gg.standard_normal((120, 25)) @ gg.standard_normal((25, 90))
    res = rs.rand_lupp_adaptive(b_exact, 8, 1e-9, rs.SketchSpec("sparsesign", 90, 8, zeta=4), rs.RngStream(85))
    assert res.rank == int(ga["rank"]) and res.status == str(ga["status"])
    assert np.array_equal(res.row_idx[: res.rank - 8], ga["row_idx"][: res.rank - 8])
    tr = np.array([[r.k, r.e_schur] for r in res.trace])
    # the last entry is at rounding level (exact-rank input): absolute floor 1e-12 x the first
    np.testing.assert_allclose(tr, ga["trace"], rtol=1e-9, atol=1e-12 * ga["trace"][0, 1])


@pytest.mark.parametrize("b,zeta", [(32, 8), (64, 4)])
def test_adaptive_sparse_sign_vs_oracle(b, zeta):
    """The sparse-sign adaptive loop at 1500 x 1200 against the oracle's (pinned to the
    reference's golden sparse-sign case): with Y_t bitwise the reference's, rank, status and
    pivots match exactly; the trace to 1e-9 relative."""
    rs = _rs()
    a, _ = orc.gen_fast_decay(1500, 1200, 1e-12, 3, 77)
    tau = 1e-8 * np.linalg.norm(a)
    ref = orc.rand_lupp_adaptive(a, b, tau, 11, zeta=zeta)
    got = rs.rand_lupp_adaptive(a, b, tau, rs.SketchSpec("sparsesign", 1200, b, zeta=zeta), rs.RngStream(11))
    assert got.rank == ref["rank"] and got.status == ref["status"] and got.rank > 2 * b
    assert np.array_equal(got.row_idx, ref["row_idx"])
    tr = np.array([[r.k, r.e_schur] for r in got.trace])
    np.testing.assert_allclose(tr, np.array(ref["trace"]), rtol=1e-9, atol=1e-12 * np.linalg.norm(a))
