"""The reference's sketching tests (`tests/test_sketching.py`) against this package: stream
and spec logic and operator construction on the host (CPU suite); applying operators runs on
the device (`gpu` marker)."""

import numpy as np
import pytest

import paper_2310_09417_b200 as rs
from paper_2310_09417_b200.errors import DimensionError

gpu = pytest.mark.gpu


def mc_mean_sq_norm(x, kind, ell, draws, seed, zeta=8):
    """Monte-Carlo oracle: mean of ||x @ Omega||_F^2 over independent draws (reference helper)."""
    spec = rs.SketchSpec(kind, n=x.shape[1], ell=ell, zeta=zeta)
    base = rs.RngStream(seed)
    total = 0.0
    for i in range(draws):
        op = rs.make_sketch(spec, base.child(i))
        total += np.linalg.norm(np.asarray(rs.apply_sketch(x, op))) ** 2
    return total / draws


# ------------------------------------------------------------------ host ---
def test_stream_determinism_and_children():
    r = rs.RngStream(123, 4)
    assert np.array_equal(r.generator().standard_normal(8), rs.RngStream(123, 4).generator().standard_normal(8))
    assert r.child(0) != r.child(1)
    assert r.child(2) == r.child(2)


def test_distinct_streams_uncorrelated():
    spec = rs.SketchSpec("gaussian", n=100, ell=100, scale="unit")
    a = np.asarray(rs.make_gaussian(spec, rs.RngStream(7, 0))).ravel()
    b = np.asarray(rs.make_gaussian(spec, rs.RngStream(7, 1))).ravel()
    assert abs(np.corrcoef(a, b)[0, 1]) < 4.0 / np.sqrt(100 * 100)


def test_spec_validation_reference_cases():
    with pytest.raises(ValueError):
        rs.SketchSpec("fourier", n=8, ell=4)
    with pytest.raises(DimensionError):
        rs.SketchSpec("gaussian", n=8, ell=9)
    with pytest.raises(DimensionError):
        rs.SketchSpec("sparsesign", n=16, ell=4, zeta=8)
    with pytest.raises(ValueError):
        rs.SketchSpec("gaussian", n=8, ell=4, scale="cubed")


def test_gaussian_mean_determinism_and_scale():
    omega = np.asarray(rs.make_gaussian(rs.SketchSpec("gaussian", n=1000, ell=1000, scale="unit"), rs.RngStream(0)))
    assert abs(omega.mean()) < 4.0 / np.sqrt(1000 * 1000)
    spec = rs.SketchSpec("gaussian", n=32, ell=8)
    assert np.array_equal(np.asarray(rs.make_gaussian(spec, rs.RngStream(5, 17))),
                          np.asarray(rs.make_gaussian(spec, rs.RngStream(5, 17))))
    a = np.asarray(rs.make_gaussian(rs.SketchSpec("gaussian", n=64, ell=16, scale="unit"), rs.RngStream(3)))
    b = np.asarray(rs.make_gaussian(rs.SketchSpec("gaussian", n=64, ell=16, scale="inv_sqrt_ell"), rs.RngStream(3)))
    assert np.allclose(a / np.sqrt(16.0), b, rtol=1e-15, atol=0)


@gpu  # to_dense materialises the operator on the device
def test_srtt_orthogonal_and_deterministic():
    op = rs.make_srtt(rs.SketchSpec("srtt", n=64, ell=64), rs.RngStream(21))
    dense = np.asarray(op.to_dense())
    assert np.linalg.norm(dense.T @ dense - np.eye(64)) <= 1e-10 * 64
    spec = rs.SketchSpec("srtt", n=32, ell=8)
    assert np.array_equal(np.asarray(rs.make_srtt(spec, rs.RngStream(1, 2)).to_dense()),
                          np.asarray(rs.make_srtt(spec, rs.RngStream(1, 2)).to_dense()))


@gpu
def test_sparse_sign_counts_and_saturation():
    op = rs.make_sparse_sign(rs.SketchSpec("sparsesign", n=50, ell=16, zeta=8), rs.RngStream(4))
    dense = np.asarray(op.to_dense())
    assert np.all((dense != 0).sum(axis=1) == 8)
    assert all(len(set(row)) == 8 for row in np.asarray(op.idx))
    op = rs.make_sparse_sign(rs.SketchSpec("sparsesign", n=20, ell=6, zeta=6), rs.RngStream(5))
    assert np.allclose(np.abs(np.asarray(op.to_dense())), 1.0 / np.sqrt(6.0), rtol=1e-15, atol=0)


# ---------------------------------------------------------------- device ---
@gpu
def test_srtt_zero_and_dense_materialization():
    op = rs.make_srtt(rs.SketchSpec("srtt", n=32, ell=8), rs.RngStream(2))
    assert np.abs(np.asarray(rs.apply_sketch(np.zeros((5, 32)), op))).max() == 0.0
    a = np.random.default_rng(3).standard_normal((7, 48))
    op = rs.make_srtt(rs.SketchSpec("srtt", n=48, ell=12), rs.RngStream(9))
    assert np.abs(np.asarray(rs.apply_sketch(a, op)) - a @ np.asarray(op.to_dense())).max() <= 1e-12


@gpu
def test_sparse_sign_matches_dense_product():
    a = np.random.default_rng(6).standard_normal((9, 40))
    op = rs.make_sparse_sign(rs.SketchSpec("sparsesign", n=40, ell=12, zeta=5), rs.RngStream(8))
    assert np.abs(np.asarray(rs.apply_sketch(a, op)) - a @ np.asarray(op.to_dense())).max() <= 1e-13


@gpu
@pytest.mark.parametrize("kind,n,ell,hot,seed,lo,hi", [("gaussian", 32, 8, 0, 11, 0.95, 1.05),
                                                        ("srtt", 256, 64, 3, 13, 0.9, 1.1),
                                                        ("sparsesign", 64, 16, 9, 17, 0.9, 1.1)])
def test_unbiased_unit_row(kind, n, ell, hot, seed, lo, hi):
    x = np.zeros((1, n))
    x[0, hot] = 1.0
    assert lo <= mc_mean_sq_norm(x, kind, ell=ell, draws=10_000, seed=seed) <= hi


@gpu
def test_apply_reference_cases():
    a = np.random.default_rng(7).standard_normal((5, 6))
    assert np.abs(np.asarray(rs.apply_sketch(a, np.eye(6))) - a).max() <= 1e-15
    u = np.arange(1.0, 9.0)[:, None]
    a = u @ np.random.default_rng(8).standard_normal((1, 30))
    y = np.asarray(rs.apply_sketch(a, rs.make_sketch(rs.SketchSpec("gaussian", n=30, ell=5), rs.RngStream(10))))
    assert np.abs(y - u @ (y[0] / u[0, 0])[None, :]).max() <= 1e-12
    a = np.random.default_rng(9).standard_normal((12, 7))
    gamma = np.asarray(rs.make_gaussian(rs.SketchSpec("gaussian", n=12, ell=4), rs.RngStream(11)))
    assert np.abs(np.asarray(rs.apply_sketch(a, gamma, side="transposed_right")) - a.T @ gamma).max() <= 1e-13
    op = rs.make_sketch(rs.SketchSpec("gaussian", n=30, ell=5), rs.RngStream(1))
    with pytest.raises(DimensionError):
        rs.apply_sketch(np.ones((4, 29)), op)
    with pytest.raises(DimensionError):
        rs.apply_sketch(np.ones((4, 29)), np.ones((28, 3)))


@gpu
def test_fixed_matrix_isometry_all_kinds():
    x = np.random.default_rng(12).standard_normal((8, 64))
    nx2 = np.linalg.norm(x) ** 2
    for kind in ("gaussian", "srtt", "sparsesign"):
        assert 0.9 <= mc_mean_sq_norm(x, kind, ell=16, draws=2_000, seed=23) / nx2 <= 1.1, kind
