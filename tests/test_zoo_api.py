"""The reference's generator tests (`tests/test_zoo.py:13-90`) against this package's zoo
(host generators on CPU; the LU-based ones on the device)."""

import numpy as np
import pytest

import paper_2310_09417_b200 as rs
from paper_2310_09417_b200.errors import DimensionError


def test_fast_decay_endpoints_orthonormal_deterministic_and_wide():
    _, sigma = rs.gen_fast_decay(50, 30, 1e-16, rs.RngStream(0))
    assert sigma[0] == 1.0 and sigma[-1] == 1e-16
    a, sigma = rs.gen_fast_decay(30, 20, 1.0, rs.RngStream(2))
    assert np.allclose(sigma, np.ones(20))
    assert np.linalg.norm(a.T @ a - np.eye(20)) <= 1e-12 * 20
    a1, _ = rs.gen_fast_decay(25, 25, 1e-8, rs.RngStream(3))
    a2, _ = rs.gen_fast_decay(25, 25, 1e-8, rs.RngStream(3))
    assert np.array_equal(a1, a2)
    with pytest.raises(DimensionError):
        rs.gen_fast_decay(10, 20, 1e-8, rs.RngStream(4))


def test_fast_decay_svd_matches_returned_sigma():
    a, sigma = rs.gen_fast_decay(60, 40, 1e-12, rs.RngStream(1))
    computed = np.linalg.svd(a, compute_uv=False)
    assert np.allclose(computed, sigma, rtol=1e-10, atol=1e-10 * sigma[0])


def test_kahan_entries_scaling_and_validation():
    zeta = 0.99
    a = rs.gen_kahan(3, zeta)
    phi = np.sqrt(1 - zeta ** 2)
    assert a[0, 0] == 1.0 and a[2, 2] == pytest.approx(zeta ** 2)
    d = np.diag([1.0, zeta, zeta ** 2])
    k = np.array([[1, -phi, -phi], [0, 1, -phi], [0, 0, 1.0]])
    assert np.abs(a - d @ k).max() <= 1e-16
    a = rs.gen_kahan(64, 0.9)
    assert a[63, 63] == pytest.approx(0.9 ** 63)
    assert np.all(np.tril(a, -1) == 0.0)
    with pytest.raises(ValueError):
        rs.gen_kahan(4, 1.0)


def test_chan_small_pattern():
    assert np.array_equal(rs.gen_chan(2), [[1.0, 1.0], [-1.0, 1.0]])
    a4 = rs.gen_chan(4)
    assert np.array_equal(a4[:, -1], np.ones(4))
    assert np.array_equal(np.tril(a4, -1)[:, :-1], np.tril(-np.ones((4, 3)), -1))
    assert np.array_equal(np.diagonal(a4), np.ones(4))


@pytest.mark.gpu
def test_chan_growth_and_no_pivoting_on_device():
    f = rs.lupp(rs.gen_chan(10))
    assert np.abs(f.U).max() / np.abs(rs.gen_chan(10)).max() == 2.0 ** 9
    assert np.array_equal(rs.lupp(rs.gen_chan(12)).perm, np.arange(12))
