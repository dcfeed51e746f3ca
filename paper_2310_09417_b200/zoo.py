"""Synthetic test matrices of the reference (`zoo.py:36-104`) and of the
benchmark configs -- input generation, not the skeleton path.

`gen_fast_decay` (Haar bases from LAPACK QR) is built on the host with numpy
exactly as the reference builds it, so a caller switching packages gets
bit-identical inputs.  `gen_kahan` / `gen_chan` with ``device=True`` and the
two config generators below are built in HBM by librskel kernels (gen.cu);
the oracle restates each in numpy with the same rounding:

* `gen_fast_decay_hadamard` (cfg5): the fast-decay spectrum
  with randomized-Hadamard bases, A = (H S0 H S1) diag(d) (S3 H S2 H),
  H the normalized Walsh-Hadamard matrix, S_i random sign diagonals --
  O(n^2 log n) on the device instead of two n x n QRs on the host;
* `gen_nonneg_lowrank` (cfg3): W H + eta N with W, H, N uniform [0, 1) from
  Philox streams (bit-identical to numpy's `Generator(Philox).random`),
  ``||eta N||_F = rel_noise ||W H||_F``, optionally rounded to fp32.
"""

import numpy as np

from .errors import DimensionError

__all__ = ["gen_fast_decay", "gen_kahan", "gen_chan", "gen_fast_decay_hadamard", "gen_nonneg_lowrank"]


def _to(a, device):
    if not device:
        return a
    from . import _device

    import torch

    return torch.as_tensor(a).to(_device.device())


def _haar(g, m, n):
    q, r = np.linalg.qr(g.standard_normal((m, n)))
    s = np.sign(np.diagonal(r))
    s[s == 0] = 1.0
    return q * s


def gen_fast_decay(m, n, beta, rng, device=False):
    """``u diag(d) v.T`` with Haar-orthonormal u (m x n), v (n x n) and
    ``d_i = beta^((i-1)/(n-1))``; returns ``(a, d)`` (reference `zoo.py:45-75`)."""
    if m < n or n < 1:
        raise DimensionError(f"need m >= n >= 1, got {m} x {n}")
    if not 0 < beta <= 1:
        raise ValueError(f"beta must be in (0, 1], got {beta}")
    g = rng.generator()
    u = _haar(g, m, n)
    v = _haar(g, n, n)
    d = np.ones(1) if n == 1 else beta ** (np.arange(n) / (n - 1))
    return _to((u * d) @ v.T, device), d


def gen_kahan(n, zeta=0.99, device=False):
    """Kahan's ``diag(zeta^i) (I - phi * strict upper ones)``, ``phi = sqrt(1 - zeta^2)``
    (reference `zoo.py:78-88`); ``device=True`` builds it in HBM (rs_kahan)."""
    if not 0 < zeta < 1:
        raise ValueError(f"zeta must be in (0, 1), got {zeta}")
    phi = np.sqrt(1.0 - zeta * zeta)
    rowpow = zeta ** np.arange(n)
    if device:
        import torch

        from . import _device, _lib

        a = torch.empty((n, n), dtype=torch.float64, device=_device.device())
        rp = torch.from_numpy(rowpow).to(a.device)
        _lib.call("rs_kahan", a.data_ptr(), n, n, rp.data_ptr(), float(0.0 - phi * 1.0), _device.stream_handle())
        return a
    k = np.eye(n) - phi * np.triu(np.ones((n, n)), 1)
    return rowpow[:, None] * k


def gen_chan(n, device=False):
    """Growth-factor matrix: unit lower triangle with -1 below the diagonal
    and a last column of ones (partial pivoting growth 2^(n-1), reference
    `zoo.py:91-104`); ``device=True`` builds it in HBM (rs_chan)."""
    if n < 1:
        raise DimensionError(f"n must be >= 1, got {n}")
    if device:
        import torch

        from . import _device, _lib

        a = torch.empty((n, n), dtype=torch.float64, device=_device.device())
        _lib.call("rs_chan", a.data_ptr(), n, n, _device.stream_handle())
        return a
    a = np.eye(n) - np.tril(np.ones((n, n)), -1)
    a[:, -1] = 1.0
    return a


def hadamard_factors(n, beta, rng):
    """Host-side parameters of `gen_fast_decay_hadamard`: the four sign
    vectors (from ``rng.generator()``) and the spectrum d."""
    if n < 1 or n & (n - 1):
        raise DimensionError(f"n must be a power of two, got {n}")
    if not 0 < beta <= 1:
        raise ValueError(f"beta must be in (0, 1], got {beta}")
    signs = rng.generator().integers(0, 2, size=(4, n)).astype(np.float64) * 2.0 - 1.0
    d = np.ones(1) if n == 1 else beta ** (np.arange(n) / (n - 1))
    return signs, d


def gen_fast_decay_hadamard(n, beta, rng, device=True):
    """n x n (n a power of two) matrix with singular values exactly
    ``d_i = beta^((i-1)/(n-1))`` and randomized-Hadamard singular vectors:
    ``A = (H S0 H S1) diag(d) (S3 H S2 H)``.  Built in HBM by four
    Walsh-Hadamard passes (rs_hadamard_init + 3 x rs_fwht_rows); returns
    ``(a, d)`` with ``a`` a CUDA tensor (``device=False``: numpy copy)."""
    import torch

    from . import _device, _lib

    signs, d = hadamard_factors(n, beta, rng)
    dev = _device.device()
    c = 1.0 / np.sqrt(n)
    mid = signs[3] * d * signs[1]          # S1 D S3 (sign flips are exact)
    rs = [torch.from_numpy(np.ascontiguousarray(v)).to(dev) for v in (signs[2], mid, signs[0])]
    x = torch.empty((n, n), dtype=torch.float64, device=dev)
    st = _device.stream_handle()
    _lib.call("rs_hadamard_init", x.data_ptr(), n, n, c, rs[0].data_ptr(), st)   # S2 (c H)
    _lib.call("rs_fwht_rows", x.data_ptr(), n, n, c, rs[1].data_ptr(), st)       # S1 D S3 (c H) ...
    _lib.call("rs_fwht_rows", x.data_ptr(), n, n, c, rs[2].data_ptr(), st)       # S0 (c H) ...
    _lib.call("rs_fwht_rows", x.data_ptr(), n, n, c, None, st)                   # (c H) ...
    if not device:
        return x.cpu().numpy(), d
    return x, d


def gen_nonneg_lowrank(m, n, r, rel_noise, rng, dtype="float32", device=True):
    """cfg3's non-negative low-rank-plus-noise matrix: ``W H + eta N`` with
    W (m x r), H (r x n), N (m x n) uniform [0, 1) drawn from
    ``rng.child(0..2)`` (numpy ``Generator(Philox).random`` bits),
    ``eta = rel_noise ||W H||_F / ||N||_F``, rounded to ``dtype``."""
    import torch

    from . import _device, _lib

    dev = _device.device()
    st = _device.stream_handle()

    def uniform(i, rows, cols):
        out = torch.empty((rows, cols), dtype=torch.float64, device=dev)
        k0, k1 = rng.child(i).philox_key()
        _lib.call("rs_uniform", k0, k1, rows * cols, out.data_ptr(), st)
        return out

    w, h = uniform(0, m, r), uniform(1, r, n)
    low = _device.dgemm(_device.Matrix(w, m, r, r, False, "torch_cuda"), _device.Matrix(h, r, n, n, False, "torch_cuda"))
    del w, h
    noise = uniform(2, m, n)
    e2 = torch.empty(2, dtype=torch.float64, device=dev)
    ws = _device.workspace().data_ptr()
    _lib.call("rs_sumsq", low.data_ptr(), n, m, n, e2[0:1].data_ptr(), ws, st)
    _lib.call("rs_sumsq", noise.data_ptr(), n, m, n, e2[1:2].data_ptr(), ws, st)
    nl, nn = (float(v) for v in e2.cpu())
    eta = rel_noise * np.sqrt(nl) / np.sqrt(nn)
    if dtype == "float32":
        out = torch.empty((m, n), dtype=torch.float32, device=dev)
        _lib.call("rs_axpy_cast", low.data_ptr(), noise.data_ptr(), float(eta), m * n, None, out.data_ptr(), st)
    else:
        out = torch.empty((m, n), dtype=torch.float64, device=dev)
        _lib.call("rs_axpy_cast", low.data_ptr(), noise.data_ptr(), float(eta), m * n, out.data_ptr(), None, st)
    if not device:
        return out.cpu().numpy()
    return out
