"""SRTT embedding as a fast transform on the device (`rs_srtt_apply`: per-row DCT-II
through one real FFT) against the reference's `SrttSketch.apply` (`sketching.py:147-155`),
restated by the oracle with scipy's DCT (pinned bitwise to the reference's golden y/yt).
FFT and pocketfft orders differ: the bar is 1e-13 relative to the row norm of A."""
import ctypes

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

import randskel_oracle as orc  # noqa: E402


def _rs():
    import paper_2310_09417_b200 as rs
    return rs


def _check(got, want, a):
    scale = np.linalg.norm(a, axis=1).max()
    assert np.abs(got - want).max() <= 1e-13 * scale, np.abs(got - want).max() / scale


@pytest.mark.parametrize("m,n,ell,layout", [
    (1, 1, 1, "row"), (3, 2, 2, "row"), (50, 997, 300, "row"), (64, 1024, 256, "col"), (40, 4096, 4096, "row"),
    (9, 30011, 512, "row"), (7, 30011, 600, "col"), (300, 2000, 1000, "row"),
])
def test_fft_path_vs_oracle(m, n, ell, layout):
    """Odd / even / prime n, ell = n, rows longer than the staged-row limit, both layouts."""
    import torch

    from paper_2310_09417_b200 import _device, sketching

    gen = np.random.default_rng(m + n)
    a = gen.standard_normal((m, n)) * np.exp(gen.standard_normal((m, n)))
    perm, signs, cols, scale = orc.srtt_operator(5, m, n, ell)
    want = orc.srtt_apply(a, perm, signs, cols, scale)
    src = torch.as_tensor(a if layout == "row" else np.asfortranarray(a)).cuda()
    got = _device.srtt_apply(_device.as_matrix(src), perm, signs, cols, scale).cpu().numpy()
    _check(got, want, a)
    op = sketching.SrttSketch(perm, signs, cols, scale)
    if ell >= sketching.SRTT_FFT_MIN_ELL:  # the operator API takes the FFT form at this width
        _check(op.apply(a), want, a)
        _check(_rs().apply_sketch(a, op), want, a)


def test_small_workspace_batches_rows():
    """A workspace of three rows: the rows go through cuFFT in batches, same result."""
    import torch

    from paper_2310_09417_b200 import _device, _lib

    lib = _lib.load()
    m, n, ell = 20, 777, 100
    a = torch.randn(m, n, dtype=torch.float64, device="cuda")
    perm, signs, cols, scale = orc.srtt_operator(9, 0, n, ell)
    dev = a.device
    pd = torch.as_tensor(perm.astype(np.int64)).to(dev)
    sd = torch.as_tensor(signs).to(dev)
    cd = torch.as_tensor(cols.astype(np.int64)).to(dev)
    y = torch.empty(m, ell, dtype=torch.float64, device=dev)
    nb = int(lib.rs_srtt_workspace_bytes(3, n))
    ws = torch.empty(nb, dtype=torch.uint8, device=dev)
    st = lib.rs_srtt_apply(m, n, ell, ctypes.c_void_p(a.data_ptr()), n, 0, ctypes.c_void_p(pd.data_ptr()),
                           ctypes.c_void_p(sd.data_ptr()), ctypes.c_void_p(cd.data_ptr()), scale,
                           ctypes.c_void_p(y.data_ptr()), ell, ctypes.c_void_p(ws.data_ptr()), nb,
                           ctypes.c_void_p(_device.stream_handle()))
    assert st == 0
    an = a.cpu().numpy()
    _check(y.cpu().numpy(), orc.srtt_apply(an, perm, signs, cols, scale), an)
    assert lib.rs_srtt_apply(m, n, ell, ctypes.c_void_p(a.data_ptr()), n, 0, ctypes.c_void_p(pd.data_ptr()),
                             ctypes.c_void_p(sd.data_ptr()), ctypes.c_void_p(cd.data_ptr()), scale,
                             ctypes.c_void_p(y.data_ptr()), ell, ctypes.c_void_p(ws.data_ptr()), 8,
                             ctypes.c_void_p(_device.stream_handle())) != 0  # less than one row: refused


def test_fft_and_dense_forms_agree():
    """The operator's two device forms (FFT, dense embedding) agree to rounding."""
    rs = _rs()
    from paper_2310_09417_b200 import _device

    op = rs.make_sketch(rs.SketchSpec("srtt", 3000, 512), rs.RngStream(4))
    a = np.random.default_rng(1).standard_normal((200, 3000))
    A = _device.as_matrix(a)
    fft = _device.srtt_apply(A, op.perm, op.signs, op.cols, op.scale).cpu().numpy()
    dense = _device.sketch_dev(A, op.device_dense()).cpu().numpy()
    _check(fft, dense, a)


def test_invalid_operator_indices_raise():
    """Out-of-range permutation / sampled-column indices raise IndexError as numpy's
    indexing does in the reference; negative indices wrap as in numpy."""
    from paper_2310_09417_b200 import _device, sketching

    n, ell = 600, 520
    perm, signs, cols, scale = orc.srtt_operator(3, 0, n, ell)
    a = np.random.default_rng(2).standard_normal((10, n))
    bad = cols.copy()
    bad[3] = n
    with pytest.raises(IndexError):
        sketching.SrttSketch(perm, signs, bad, scale).apply(a)
    neg = cols.copy()
    neg[4] = neg[4] - n
    want = orc.srtt_apply(a, perm, signs, cols, scale)
    got = _device.srtt_apply(_device.as_matrix(a), perm, signs, neg, scale).cpu().numpy()
    _check(got, want, a)
