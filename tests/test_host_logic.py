"""Host-side logic that needs no GPU: RNG streams, specs, argument checks."""

import numpy as np
import pytest

import paper_2310_09417_b200 as rs
import randskel_oracle as orc
from paper_2310_09417_b200 import _omega


def test_child_streams_match_oracle():
    r = rs.RngStream(123, 4)
    for i in (0, 1, 7, 1 << 40, 1 << 41):
        assert r.child(i).stream == orc.child_stream(4, i)
    assert r.child(2) == r.child(2) and r.child(0) != r.child(1)


def test_make_gaussian_bitwise_equals_oracle_draw():
    spec = rs.SketchSpec("gaussian", n=300, ell=17)
    om = rs.make_gaussian(spec, rs.RngStream(5, 9))
    assert np.array_equal(om, orc.gaussian(5, 9, 300, 17))
    unit = rs.make_gaussian(spec.__class__("gaussian", 300, 17, scale="unit"), rs.RngStream(5, 9))
    assert np.array_equal(unit, orc.gaussian(5, 9, 300, 17, unit=True))


def test_pinned_block_draw_is_bitwise_the_reference_block():
    # per-block Omega_t of the adaptive loop: child(t), variance 1/b (skeleton.py:286-295)
    rng = rs.RngStream(0)
    h = _omega.draw_block_pinned(500, 64, rng.child(3), unit_scale=False) if _pinned_ok() else None
    ref = orc.gaussian(0, orc.child_stream(0, 3), 500, 64)
    if h is not None:
        assert np.array_equal(h.numpy(), ref)
    g = rng.child(3).generator()
    buf = np.empty((500, 64))
    g.standard_normal(out=buf)
    buf /= np.sqrt(64)
    assert np.array_equal(buf, ref)


def _pinned_ok():
    import torch

    return torch.cuda.is_available()


def test_spec_validation():
    with pytest.raises(ValueError):
        rs.SketchSpec("fourier", n=8, ell=4)
    with pytest.raises(rs.DimensionError):
        rs.SketchSpec("gaussian", n=8, ell=9)
    with pytest.raises(rs.DimensionError):
        rs.SketchSpec("sparsesign", n=16, ell=4, zeta=8)
    with pytest.raises(ValueError):
        rs.SketchSpec("gaussian", n=8, ell=4, scale="cubed")


def test_argument_errors_raised_before_device_use():
    a = np.eye(10)
    spec = rs.SketchSpec("gaussian", 10, 2)
    with pytest.raises(ValueError):
        rs.rand_lupp_adaptive(a, 2, 0.0, spec, rs.RngStream(0))
    with pytest.raises(rs.DimensionError):
        rs.rand_lupp_adaptive(a, 11, 1.0, spec, rs.RngStream(0))
    with pytest.raises(rs.DimensionError):
        rs.rand_lupp(a, 0, spec, rs.RngStream(0))
    with pytest.raises(rs.DimensionError):
        rs.column_id(a, 11, spec, rs.RngStream(0))
    with pytest.raises(rs.DimensionError):
        rs.rand_lupp_adaptive(np.ones(5), 1, 1.0, spec, rs.RngStream(0))


def test_no_cpu_fallback():
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(rs.DeviceError):
        rs.rand_lupp_adaptive(np.eye(10), 2, 1.0, rs.SketchSpec("gaussian", 10, 2), rs.RngStream(0))


def test_error_trace_requires_increasing_ranks():
    tr = rs.ErrorTrace()
    tr.append(rs.TraceRecord(k=10, e_schur=1.0))
    with pytest.raises(ValueError):
        tr.append(rs.TraceRecord(k=10, e_schur=0.5))


def test_philox_key_matches_numpy_conversion():
    """RngStream.philox_key() = the key numpy actually uses (float64 rounding
    of a word >= 2**63 when the other word is small)."""
    import numpy as np
    import paper_2310_09417_b200 as rs

    for seed, stream in [(0, 0), (0, 0xa706dd2f4d197e6f), (1 << 63, 1 << 63), (5, (1 << 64) - 1), (2**62, 7)]:
        s = rs.RngStream(seed, stream)
        k = np.random.Philox(key=[seed, stream]).state["state"]["key"]
        assert s.philox_key() == (int(k[0]), int(k[1]))
    assert rs.RngStream(0, 0xa706dd2f4d197e6f).philox_key()[1] != 0xa706dd2f4d197e6f


def test_zoo_generators_match_reference_construction():
    """gen_fast_decay / gen_kahan / gen_chan build the reference's matrices
    bit for bit (the oracle restates `zoo.py:36-104`)."""
    import os
    import sys

    import numpy as np
    import paper_2310_09417_b200 as rs

    sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle"))
    import randskel_oracle as orc

    a, d = rs.gen_fast_decay(60, 40, 1e-6, rs.RngStream(7, 3))
    a2, d2 = orc.gen_fast_decay(60, 40, 1e-6, 7, 3)
    assert np.array_equal(a, a2) and np.array_equal(d, d2)
    assert np.array_equal(rs.gen_kahan(30, 0.9), orc.gen_kahan(30, 0.9))
    assert np.array_equal(rs.gen_chan(12), orc.gen_chan(12))
    import pytest

    with pytest.raises(rs.DimensionError):
        rs.gen_fast_decay(3, 5, 0.5, rs.RngStream(0))
    with pytest.raises(ValueError):
        rs.gen_kahan(4, 1.5)


def test_host_prefault_result_buffer():
    """HostPrefault: pages populated in the background up to advance(), the result a
    contiguous writeable zero-filled array over the mapping; close is idempotent."""
    from paper_2310_09417_b200._device import HostPrefault

    hp = HostPrefault(64 << 20)
    hp.advance(10 << 20)
    hp.advance(5 << 20)  # never moves back
    a = hp.array((1000, 1000), np.float64)
    assert a.flags.c_contiguous and a.flags.writeable and a.shape == (1000, 1000)
    assert not a.any()
    a[:] = 3.0
    assert a.sum() == 3.0e6
    hp.close()
    big = HostPrefault(1 << 20).array((1000, 1000), np.float64)  # larger than the mapping
    assert big.shape == (1000, 1000)
