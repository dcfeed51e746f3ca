"""Skeleton error evaluators on the device.

  row_id_error(a, result)         ||a - w a[row_idx]||_F         (`skeleton.py:542-547`)
  stable_row_id_error(a, result)  ||a.T - Q Q.T a.T||_F, Q an orthonormal basis of
                                  a[row_idx].T                   (`skeleton.py:550-562`)

Both stream A once through the DMMA GEMM in row blocks (the residual block
never exists beyond a few hundred MB) and accumulate the squared Frobenius
norm with the deterministic two-stage reduction.  The orthonormal basis of
the skeleton rows comes from their interpolative form: LUPP of a[I].T gives
a[I].T = W' a[I].T[J] with sigma_min(W') >= 1, so CholeskyQR2 of W' is
stable and spans the same space (Q Q.T is the same projector as the
reference's unpivoted-QR Q when a[I] has full row rank).
"""

import math

import torch

from . import _device, _engine, _lib, dense
from .errors import NumericalError

__all__ = ["row_id_error", "stable_row_id_error"]

_ROW_BLOCK = 8192


def _st():
    return _device.stream_handle()


def _idx(x):
    if isinstance(x, torch.Tensor):
        return x.to(device=_device.device(), dtype=torch.int64)
    import numpy as np

    return torch.as_tensor(np.asarray(x, dtype=np.int64)).to(_device.device())


def _sumsq_add(X, acc):
    """acc += ||X||_F^2 (X row-major Matrix), fixed order."""
    part = torch.empty(1, dtype=torch.float64, device=acc.device)
    _lib.call("rs_sumsq", X.ptr, X.ld, X.rows, X.cols, part.data_ptr(), _device.workspace().data_ptr(), _st())
    acc.add_(part)


def _residual_norm(A, L, Rt_rows, ridx=None):
    """||A - L R||_F with L (m x k) row-major and R given as its rows
    (Rt_rows: row-major k x n, optionally gathered by ridx), in row blocks."""
    m, n = A.shape
    dev = _device.device()
    acc = torch.zeros(1, dtype=torch.float64, device=dev)
    Ar = A.row_major()
    for r0 in range(0, m, _ROW_BLOCK):
        rows = min(_ROW_BLOCK, m - r0)
        E = torch.empty((rows, n), dtype=torch.float64, device=dev)
        dense._gemm(dense._mat(E), L.sub(r0, 0, rows, L.cols), Rt_rows, alpha=-1.0, beta=1.0,
                    Cin=Ar.sub(r0, 0, rows, n), bidx=ridx)
        _sumsq_add(dense._mat(E), acc)
    return math.sqrt(float(acc.item()))


def row_id_error(a, result):
    """Plain row-ID residual ``||a - w @ a[row_idx]||_F`` (reference `skeleton.py:542-547`)."""
    if result.row_idx is None or result.w is None:
        raise ValueError("result carries no row skeletons")
    A = _device.as_matrix(a, "a")
    W = _device.as_matrix(result.w, "w").row_major()
    ridx = _idx(result.row_idx)
    return _residual_norm(A, W, A.row_major(), ridx=ridx)


def _orthonormal_basis(B):
    """Q (n x k, row-major) with orthonormal columns spanning range(B), B an
    n x k device Matrix of full column rank."""
    n, k = B.shape
    dev = _device.device()
    st, Wp, fail = _engine.factor_sample(B.row_major(), want_w=True)
    if fail is not None:
        raise NumericalError(f"skeleton rows are exactly rank deficient (step {fail})")
    Q = dense._mat(Wp)
    status = torch.empty(1, dtype=torch.int32, device=dev)
    for _ in range(2):  # CholeskyQR2
        G = torch.empty((k, k), dtype=torch.float64, device=dev)
        dense._gemm(dense._mat(G), Q.T, Q)
        _lib.call("rs_cholesky", G.data_ptr(), k, k, status.data_ptr(), _st())
        if int(status.item()) != 0:
            raise NumericalError("Gram matrix of the skeleton basis is not positive definite")
        # Q <- Q R^{-1}:  R^T Q^T = Q^T
        Qt = dense._trsm_left(dense._mat(G).T, Q.T.row_major(), lower=True, unit=False)
        Q = Qt.T.row_major()
    return Q


def stable_row_id_error(a, result):
    """Projection residual ``||a.T - Q Q.T a.T||_F`` through an orthonormal
    basis of the skeleton rows (reference `skeleton.py:550-562`)."""
    if result.row_idx is None:
        raise ValueError("result carries no row skeletons")
    A = _device.as_matrix(a, "a")
    m, n = A.shape
    ridx = _idx(result.row_idx)
    Ar = A.row_major()
    B = dense._mat(_gather_rows(Ar, ridx)).T        # a[I].T : n x k
    Q = _orthonormal_basis(B)                        # n x k
    k = Q.cols
    AQ = torch.empty((m, k), dtype=torch.float64, device=_device.device())
    dense._gemm(dense._mat(AQ), Ar, Q)               # A Q   (m x k)
    # ||A.T - Q Q.T A.T||_F = ||A - (A Q) Q.T||_F
    return _residual_norm(A, dense._mat(AQ), Q.T.row_major())


def _gather_rows(Ar, idx):
    out = torch.empty((idx.numel(), Ar.cols), dtype=torch.float64, device=_device.device())
    _lib.call("rs_gather_rows", Ar.ptr, Ar.ld, idx.data_ptr(), idx.numel(), Ar.cols, out.data_ptr(),
              max(Ar.cols, 1), _st())
    return out
