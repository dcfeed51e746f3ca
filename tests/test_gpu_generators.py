"""Device input generators (csrc/gen.cu, paper_2310_09417_b200.zoo) against
their numpy statements (the reference's `zoo.py:78-104` and the oracle's
restatements of the config generators): bit for bit."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

import randskel_oracle as orc  # noqa: E402


@pytest.fixture(scope="module")
def rs():
    import paper_2310_09417_b200 as rs

    return rs


@pytest.mark.parametrize("seed,stream", [(0, 0), (7, 1 << 41), (3, (1 << 64) - 1)])
def test_uniform_is_numpy_philox_random(rs, seed, stream):
    from paper_2310_09417_b200 import _device, _lib

    n = 100003
    k0, k1 = rs.RngStream(seed, stream).philox_key()
    out = torch.empty(n, dtype=torch.float64, device="cuda")
    _lib.call("rs_uniform", k0, k1, n, out.data_ptr(), _device.stream_handle())
    ref = rs.RngStream(seed, stream).generator().random(n)
    assert np.array_equal(out.cpu().numpy(), ref)


@pytest.mark.parametrize("n", [1, 2, 64, 256, 2048])
def test_hadamard_fast_decay_bitwise(rs, n):
    if n == 1:
        with pytest.raises(Exception):
            rs.gen_fast_decay_hadamard(3, 1e-16, rs.RngStream(0))
        return
    rng = rs.RngStream(5).child(1 << 41)
    a, d = rs.gen_fast_decay_hadamard(n, 1e-16, rng)
    a0, d0 = orc.gen_fast_decay_hadamard(n, 1e-16, rng.seed, rng.stream)
    assert np.array_equal(d, d0)
    assert np.array_equal(a.cpu().numpy(), a0)
    # exact spectrum up to rounding
    s = np.linalg.svd(a0, compute_uv=False)
    assert np.abs(s - d0).max() <= 1e-13


@pytest.mark.parametrize("n", [1, 7, 300])
def test_kahan_and_chan_bitwise(rs, n):
    assert np.array_equal(rs.gen_kahan(n, 0.99, device=True).cpu().numpy(), orc.gen_kahan(n, 0.99))
    assert np.array_equal(rs.gen_chan(n, device=True).cpu().numpy(), orc.gen_chan(n))


def test_nonneg_lowrank_recipe(rs):
    """cfg3's generator: uniforms bit-identical to numpy's Philox streams; the
    W H product on the DMMA GEMM, so the matrix agrees with numpy's to fp64
    rounding (and to the fp32 cast in all but rare boundary cases)."""
    m, n, r = 700, 500, 20
    rng = rs.RngStream(0).child(1 << 41)
    a = rs.gen_nonneg_lowrank(m, n, r, 1e-6, rng, dtype="float64").cpu().numpy()
    w = orc.philox_uniform(rng.child(0).seed, rng.child(0).stream, (m, r))
    h = orc.philox_uniform(rng.child(1).seed, rng.child(1).stream, (r, n))
    nz = orc.philox_uniform(rng.child(2).seed, rng.child(2).stream, (m, n))
    low = w @ h
    eta = 1e-6 * np.linalg.norm(low) / np.linalg.norm(nz)
    ref = low + eta * nz
    assert np.abs(a - ref).max() <= 1e-13 * np.abs(ref).max()
    a32 = rs.gen_nonneg_lowrank(m, n, r, 1e-6, rng).cpu().numpy()
    assert a32.dtype == np.float32 and (a32 >= 0).all()
    assert np.mean(a32 == ref.astype(np.float32)) > 0.999
