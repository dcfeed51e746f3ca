"""Device Philox4x64-10 + ziggurat standard normals vs numpy, bit for bit."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.mark.parametrize("seed,stream,n,ell", [
    (0, 0, 1000, 1), (3, 77, 4096, 256), (0, 0x123456789ABCDEF, 20000, 64),
    (12345, 1 << 40, 16384, 1024), (7, 9, 333, 17),
])
def test_device_normals_bitwise(seed, stream, n, ell):
    import paper_2310_09417_b200 as rs
    from paper_2310_09417_b200 import _device

    s = rs.RngStream(seed, stream)
    ref = s.generator().standard_normal((n, ell))
    got = _device.gaussian(s, n, ell, unit=True).cpu().numpy()
    bad = np.flatnonzero(got.view(np.uint64) != ref.view(np.uint64))
    assert bad.size == 0, (bad.size, bad[:5], got.ravel()[bad[:5]], ref.ravel()[bad[:5]])
    scaled = _device.gaussian(s, n, ell).cpu().numpy()
    assert np.array_equal(scaled, rs.make_gaussian(rs.SketchSpec("gaussian", n, ell), s))


def test_device_normals_many_streams():
    """Adaptive-loop streams (child(t)) of a 20000 x 64 block: 2.56M normals."""
    import paper_2310_09417_b200 as rs
    from paper_2310_09417_b200 import _device

    base = rs.RngStream(0)
    for t in (0, 1, 2, 117):
        s = base.child(t)
        ref = s.generator().standard_normal((20000, 64)) / np.sqrt(64)
        got = _device.gaussian(s, 20000, 64).cpu().numpy()
        assert np.array_equal(got, ref), t


@pytest.mark.parametrize("stream", [0xa706dd2f4d197e6f, (1 << 64) - 1, 1 << 63])
def test_device_normals_high_key_words(stream):
    """numpy rounds a key word >= 2**63 through float64 (np.asarray of the
    key list); the device draw must use the same words."""
    import paper_2310_09417_b200 as rs
    from paper_2310_09417_b200 import _device

    for s in (rs.RngStream(0, stream), rs.RngStream(stream, 5), rs.RngStream(stream, stream)):
        ref = s.generator().standard_normal((300, 40))
        got = _device.gaussian(s, 300, 40, unit=True).cpu().numpy()
        assert np.array_equal(got, ref)


def test_sketch_paths_device_vs_host_rng(monkeypatch):
    """rand_lupp / column_id / adaptive give identical results with the
    device draw and with RSKEL_HOST_RNG=1."""
    import paper_2310_09417_b200 as rs

    rng = np.random.default_rng(5)
    a = rng.standard_normal((700, 40)) @ rng.standard_normal((40, 500))
    spec = rs.SketchSpec("gaussian", 500, 32)
    out = {}
    for mode in ("0", "1"):
        monkeypatch.setenv("RSKEL_HOST_RNG", mode)
        r1 = rs.rand_lupp(a, 32, spec, rs.RngStream(3))
        r2 = rs.column_id(a, 32, spec, rs.RngStream(4))
        r3 = rs.rand_lupp_adaptive(a, 8, 1e-8, spec, rs.RngStream(6))
        out[mode] = (r1.row_idx, r1.w, r2.col_idx, r2.x, r3.row_idx, r3.w, r3.rank)
    for x, y in zip(out["0"], out["1"]):
        assert np.array_equal(np.asarray(x), np.asarray(y))
