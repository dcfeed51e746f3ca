"""Synthetic test matrices of the reference (`zoo.py:36-104`) -- input
generation, not the skeleton path.

They are built on the host with numpy exactly as the reference builds them
(same generator stream, same Haar construction), so a caller switching
packages gets bit-identical inputs; the skeleton routines then move them to
the device.  ``device=True`` returns a CUDA tensor instead of a numpy array.
"""

import numpy as np

from .errors import DimensionError

__all__ = ["gen_fast_decay", "gen_kahan", "gen_chan"]


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
    (reference `zoo.py:78-88`)."""
    if not 0 < zeta < 1:
        raise ValueError(f"zeta must be in (0, 1), got {zeta}")
    phi = np.sqrt(1.0 - zeta * zeta)
    k = np.eye(n) - phi * np.triu(np.ones((n, n)), 1)
    return _to(zeta ** np.arange(n)[:, None] * k, device)


def gen_chan(n, device=False):
    """Growth-factor matrix: unit lower triangle with -1 below the diagonal
    and a last column of ones (partial pivoting growth 2^(n-1), reference
    `zoo.py:91-104`)."""
    if n < 1:
        raise DimensionError(f"n must be >= 1, got {n}")
    a = np.eye(n) - np.tril(np.ones((n, n)), -1)
    a[:, -1] = 1.0
    return _to(a, device)
