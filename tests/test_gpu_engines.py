"""Both sketch engines (int8 tensor cores by default, fp64 DMMA on request)
against the reference fixtures, and the tensor-core path's input checks."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

from conftest import golden  # noqa: E402


@pytest.fixture
def rs():
    import paper_2310_09417_b200 as rs

    yield rs
    rs.set_sketch_engine("ozaki")


@pytest.mark.parametrize("engine", ["ozaki", "dmma"])
@pytest.mark.parametrize("case", ["adapt_fd200", "adapt_b25", "adapt_exhausted", "adapt_maxrank15"])
def test_adaptive_golden_both_engines(rs, engine, case):
    rs.set_sketch_engine(engine)
    g = golden(case)
    a = g["a"]
    mr = int(g["max_rank"])
    res = rs.rand_lupp_adaptive(a, int(g["b"]), float(g["tau"]), rs.SketchSpec("gaussian", a.shape[1], int(g["b"])),
                                rs.RngStream(int(g["seed"])), max_rank=None if mr < 0 else mr)
    assert res.status == str(g["status"]) and res.rank == int(g["rank"])
    assert np.array_equal(res.row_idx, g["row_idx"])
    tr = np.array([[r.k, r.e_schur] for r in res.trace])
    assert np.abs(tr[:, 1] - g["trace"][:, 1]).max() <= 1e-12 * np.linalg.norm(a)


@pytest.mark.parametrize("engine", ["ozaki", "dmma"])
def test_fixed_rank_golden_both_engines(rs, engine):
    rs.set_sketch_engine(engine)
    a = golden("fast_decay_300")["a"]
    for k, seed in ((40, 3), (150, 2)):
        g = golden(f"rand_lupp_fd300_k{k}")
        r = rs.rand_lupp(a, k, rs.SketchSpec("gaussian", 300, 32), rs.RngStream(seed))
        assert np.array_equal(r.row_idx, g["row_idx"])
        g = golden(f"column_id_fd300_k{k}")
        c = rs.column_id(a, k, rs.SketchSpec("gaussian", 300, 32), rs.RngStream(seed))
        assert np.array_equal(c.col_idx, g["col_idx"])


@pytest.mark.parametrize("bad", [np.nan, np.inf])
def test_non_finite_input_raises(rs, bad):
    """The digit planes cannot carry NaN/inf (fmax drops NaN); the slicer flags
    them and the API raises the reference's ValueError (`dense.py:63-67`)."""
    a = np.random.default_rng(0).standard_normal((200, 150))
    a[17, 33] = bad
    spec = rs.SketchSpec("gaussian", 150, 16)
    with pytest.raises(ValueError):
        rs.rand_lupp_adaptive(a, 16, 1e-6, spec, rs.RngStream(0))
    with pytest.raises(ValueError):
        rs.rand_lupp(a, 20, spec, rs.RngStream(0))
    with pytest.raises(ValueError):
        rs.column_id(a, 20, rs.SketchSpec("gaussian", 200, 16), rs.RngStream(0))


def test_fp32_input_sketched_from_fp32_planes(rs):
    """fp32 input: 4 digit planes read from the fp32 values; the skeletons agree with the
    fp64 run on the exact upcast (well-separated spectrum)."""
    g = np.random.default_rng(5)
    a = (g.standard_normal((600, 40)) @ g.standard_normal((40, 400))).astype(np.float32)
    spec = rs.SketchSpec("gaussian", 400, 16)
    r32 = rs.rand_lupp_adaptive(a, 16, 1e-3 * np.linalg.norm(a), spec, rs.RngStream(1))
    r64 = rs.rand_lupp_adaptive(a.astype(np.float64), 16, 1e-3 * np.linalg.norm(a), spec, rs.RngStream(1))
    assert r32.rank == r64.rank and np.array_equal(r32.row_idx, r64.row_idx)


@pytest.mark.parametrize("fold", [False, True])
def test_tensor_core_tail_split_is_bitwise(rs, fold):
    """The sketch kernel halves the last partial wave's units over two CTAs and sums their
    int32 accumulators exactly (csrc/ozaki.cu `oz_item`).  Rows of a launch that splits
    (20480 x 4096: 640 units on 148 SMs, a 48-unit tail) must equal, bit for bit, the same
    rows sliced and multiplied alone (2304 rows: 72 units, no split) -- the row-local
    determinism contract of include/rskel.h."""
    import os
    import sys

    sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tools"))
    from oz_check import oz

    g = torch.Generator(device="cuda").manual_seed(11)
    M, K, N = 20480, 4096 if not fold else 1000, 64
    A = torch.randn(M, K, dtype=torch.float64, device="cuda", generator=g)
    om = torch.randn(K, N, dtype=torch.float64, device="cuda", generator=g)
    Y, _ = oz(A, False, om)
    for r0 in (0, M - 2304):  # a leading block and the block whose tiles are the split tail
        Ys, _ = oz(A[r0:r0 + 2304].contiguous(), False, om)
        assert torch.equal(Y[r0:r0 + 2304], Ys)
