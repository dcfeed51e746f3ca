"""Dense building blocks of the skeleton path on the B200 -- drop-in for the
hot-path part of `randskel.dense` (`dense.py:46-354,507-561`).

  lupp(a)                         blocked right-looking LUPP, panel 64
  lupp_blocked_step(f, new_cols)  extend factors by a block (Schur + lupp)
  triangular_solve(t, b, ...)     blocked TRSM (inverted 64x64 diagonal blocks + DMMA GEMM)
  gemm, frobenius_norm, row_permute, invert_permutation

All arithmetic runs in librskel.so (panel kernel, DMMA GEMM, trinv, gathers);
torch is used for device memory and for pure data movement (slicing,
concatenation of factor blocks).  Results come back in the caller's
container (numpy -> numpy, CUDA tensor -> CUDA tensor).
"""

import math

import numpy as np
import torch

from . import _device, _lib
from .errors import DimensionError, RankDeficientError, SingularError

__all__ = [
    "LUFactors",
    "gemm",
    "lupp",
    "lupp_blocked_step",
    "triangular_solve",
    "frobenius_norm",
    "row_permute",
    "invert_permutation",
]

PANEL = 64  # `dense.py:46`


class LUFactors:
    """``A[perm] = L @ U`` (reference `dense.py:70-93`)."""

    __slots__ = ("L", "U", "perm")

    def __init__(self, L, U, perm):
        self.L = L
        self.U = U
        self.perm = perm

    @property
    def k(self):
        return self.L.shape[1]


# ---------------------------------------------------------------- helpers --
def _ws():
    return _device.workspace().data_ptr()


def _st():
    return _device.stream_handle()


def _gemm(C, A, B, alpha=1.0, beta=0.0, Cin=None, aidx=None, bidx=None, cidx=None):
    """C = alpha A B + beta Cin on the DMMA kernel (C row-major Matrix view)."""
    if B.colmajor:
        B = B.row_major()
    if Cin is not None and Cin.colmajor:
        Cin = Cin.row_major()
    if A.colmajor and aidx is not None:
        A = A.row_major()
    M = C.rows
    _lib.call(
        "rs_dgemm", M, C.cols, A.cols, float(alpha), A.ptr, A.ld, int(A.colmajor),
        aidx.data_ptr() if aidx is not None else None, B.ptr, B.ld,
        bidx.data_ptr() if bidx is not None else None, float(beta),
        Cin.ptr if Cin is not None else None, Cin.ld if Cin is not None else 0,
        cidx.data_ptr() if cidx is not None else None, C.ptr, C.ld, _ws(), _st(),
    )
    return C


def _sumsq(X):
    X = X.row_major()
    out = torch.empty(1, dtype=torch.float64, device=X.t.device)
    _lib.call("rs_sumsq", X.ptr, X.ld, X.rows, X.cols, out.data_ptr(), _ws(), _st())
    return float(out.item())


def _check_finite(X, name="matrix"):
    if X.rows and X.cols and not math.isfinite(_sumsq(X)):
        raise ValueError(f"{name} contains non-finite entries")


def _gather_rows(X, idx, out=None):
    """out[i] = X[idx[i]] (row-major)."""
    X = X.row_major()
    n = idx.numel()
    if out is None:
        out = _device.empty(n, X.cols, X.kind)
    if n and X.cols:
        _lib.call("rs_gather_rows", X.ptr, X.ld, idx.data_ptr(), n, X.cols, out.ptr, out.ld, _st())
    return out


def _out(X, kind):
    if isinstance(X, _device.Matrix):
        X = X.tensor()
    return _device.to_output(X.contiguous() if kind != "torch_cuda" else X, kind)


def _idx_out(p, kind):
    return _device.to_host_index(p, kind)


# ------------------------------------------------------------------ lupp ----
def _lupp_device(A, allow_partial):
    """In-place blocked LUPP of the row-major device Matrix A (m x n, m >= n).
    Returns (perm (device int64), ncols).  Panel factorisation runs in the
    cooperative panel kernel on the trailing rows; the row permutation is then
    applied to whole rows (the reference's full-row swaps, `dense.py:199-202`);
    U12 = L11^{-1} A12 and A22 -= L21 U12 run on the DMMA GEMM."""
    m, n = A.shape
    dev = A.t.device
    perm = torch.arange(m, dtype=torch.int64, device=dev)
    sub = torch.empty(max(m, 1), dtype=torch.int64, device=dev)
    npanel = (n + PANEL - 1) // PANEL
    nc_dev = torch.empty(max(npanel, 1), dtype=torch.int32, device=dev)
    tmp = torch.empty(max(m * n, 1), dtype=torch.float64, device=dev)
    linv = torch.empty((PANEL, PANEL), dtype=torch.float64, device=dev)
    for bi, j0 in enumerate(range(0, n, PANEL)):
        w = min(PANEL, n - j0)
        R = m - j0
        blk = A.sub(j0, j0, R, w)
        _lib.call("rs_panel_lupp", blk.ptr, A.ld, R, w, sub.data_ptr(), nc_dev[bi:].data_ptr(), _ws(), _st())
        # physical row order = position order (full rows, like the reference's swaps)
        rows = A.sub(j0, 0, R, n)
        _lib.call("rs_gather_rows", rows.ptr, A.ld, sub.data_ptr(), R, n, tmp.data_ptr(), n, _st())
        _lib.call("rs_gather_rows", tmp.data_ptr(), n, None, R, n, rows.ptr, A.ld, _st())
        perm[j0:] = perm[j0:][sub[:R]]
        if allow_partial:  # the caller wants the factored prefix: stop at the first short panel
            nc = int(nc_dev[bi].item())
            if nc < w:
                return perm, j0 + nc
        # (without allow_partial the panel counts are read once at the end: a short panel
        # only leaves the rest unfactored, and the call raises)
        if j0 + w < n:
            # U12 = L11^{-1} A12
            L11 = A.sub(j0, j0, w, w)
            _lib.call("rs_trinv", L11.ptr, A.ld, 1, None, w, 1, 1, linv.data_ptr(), PANEL, _st())
            A12 = A.sub(j0, j0 + w, w, n - j0 - w)
            t12 = _device.Matrix(tmp, w, n - j0 - w, max(n - j0 - w, 1), False, A.kind)
            _gemm(t12, _device.Matrix(linv, w, w, PANEL, False, A.kind), A12)
            _lib.call("rs_gather_rows", t12.ptr, t12.ld, None, w, n - j0 - w, A12.ptr, A.ld, _st())
            # A22 -= L21 U12
            if j0 + w < m:
                A22 = A.sub(j0 + w, j0 + w, m - j0 - w, n - j0 - w)
                _gemm(A22, A.sub(j0 + w, j0, m - j0 - w, w), A12, alpha=-1.0, beta=1.0, Cin=A22)
    if not allow_partial and npanel:
        ncs = nc_dev[:npanel].tolist()
        for bi, nc in enumerate(ncs):
            w = min(PANEL, n - bi * PANEL)
            if nc < w:
                raise RankDeficientError(bi * PANEL + nc)
    return perm, n


def _split_lu(A, k):
    """(L, U) tensors from the in-place storage of the first k columns."""
    X = A.tensor()
    m = X.shape[0]
    L = torch.tril(X[:, :k], -1)
    L[torch.arange(k, device=X.device), torch.arange(k, device=X.device)] = 1.0
    U = torch.triu(X[:k, :k])
    return L, U


def lupp(a):
    """LU with row partial pivoting: ``a[perm] = L @ U`` (reference `dense.py:247-281`).

    Raises DimensionError (m < n), ValueError (non-finite), RankDeficientError(step).
    """
    m, n = _device.shape_of(a)
    if m < n:
        raise DimensionError(f"lupp requires rows >= cols, got {m} x {n}")
    A0 = _device.as_matrix(a)
    _check_finite(A0)
    A = A0.copy()
    perm, _ = _lupp_device(A, allow_partial=False)
    L, U = _split_lu(A, n)
    kind = A0.kind
    return LUFactors(_out(L, kind), _out(U, kind), _idx_out(perm, kind))


def _lupp_partial_device(S):
    """`_lupp_partial` (`dense.py:284-298`) on a device Matrix: (L, U, perm, ncols) tensors."""
    A = S.copy()
    perm, nc = _lupp_device(A, allow_partial=True)
    L, U = _split_lu(A, nc)
    return L, U, perm, nc


# -------------------------------------------------------- blocked extension --
def _t(x):
    """numpy / torch -> fp64 CUDA tensor (contiguous)."""
    if isinstance(x, torch.Tensor):
        return x.to(device=_device.device(), dtype=torch.float64).contiguous()
    return torch.as_tensor(np.ascontiguousarray(x, dtype=np.float64)).to(_device.device())


def _ti(x):
    if isinstance(x, torch.Tensor):
        return x.to(device=_device.device(), dtype=torch.int64)
    return torch.as_tensor(np.asarray(x, dtype=np.int64)).to(_device.device())


def _mat(t, kind="torch_cuda"):
    return _device.Matrix(t, t.shape[0], t.shape[1], max(t.shape[1], 1), False, kind)


def _solve_lower_unit(L1, B):
    """X = L1^{-1} B for unit-lower L1 (k x k) by blocked forward substitution."""
    return _trsm_left(_mat(L1), _mat(B), lower=True, unit=True)


def lupp_blocked_step(factors, new_cols):
    """Factors of ``[Y, new_cols]`` from factors of Y (reference `dense.py:301-354`)."""
    kind = _device.as_matrix(new_cols).kind if isinstance(new_cols, torch.Tensor) else "numpy"
    if factors is None or factors.k == 0:
        return lupp(new_cols)
    m0, b = _device.shape_of(new_cols)
    Lh = _t(factors.L)
    m, k = Lh.shape
    if m0 != m:
        raise DimensionError("new block row count does not match the factors")
    if k + b > m:
        raise DimensionError("extended factorization would have more cols than rows")
    Y = _mat(_t(new_cols))
    _check_finite(Y, "new_cols")
    perm = _ti(factors.perm)
    PY = _gather_rows(Y, perm)
    L1, L2 = Lh[:k].contiguous(), Lh[k:].contiguous()
    U2 = _solve_lower_unit(L1, PY.tensor()[:k].contiguous())
    S = _device.empty(m - k, b)
    _gemm(S, _mat(L2), U2, alpha=-1.0, beta=1.0, Cin=PY.sub(k, 0, m - k, b))
    sL, sU, sperm, nc = _lupp_partial_device(S)
    if nc < b:
        raise RankDeficientError(k + nc)
    L2p = L2[sperm]
    Lnew = torch.zeros((m, k + b), dtype=torch.float64, device=Lh.device)
    Lnew[:k, :k] = L1
    Lnew[k:, :k] = L2p
    Lnew[k:, k:] = sL
    Uh = _t(factors.U)
    Unew = torch.zeros((k + b, k + b), dtype=torch.float64, device=Lh.device)
    Unew[:k, :k] = Uh
    Unew[:k, k:] = U2.tensor()
    Unew[k:, k:] = sU
    pnew = perm.clone()
    pnew[k:] = perm[k:][sperm]
    return LUFactors(_out(Lnew, kind), _out(Unew, kind), _idx_out(pnew, kind))


# --------------------------------------------------------------- TRSM -------
def _trsm_left(T, B, lower, unit):
    """X = T^{-1} B (T square Matrix view, any layout; B row-major Matrix).
    Blocked substitution: 64 x 64 diagonal blocks inverted by the trinv
    kernel, off-diagonal updates on the DMMA GEMM."""
    n = T.rows
    nrhs = B.cols
    X = B.copy()
    if n == 0 or nrhs == 0:
        return X
    dev = X.t.device
    inv = torch.empty((PANEL, PANEL), dtype=torch.float64, device=dev)
    tmp = torch.empty((PANEL, nrhs), dtype=torch.float64, device=dev)
    starts = list(range(0, n, PANEL))
    if not lower:
        starts = starts[::-1]
    rs_, cs_ = (1, T.ld) if T.colmajor else (T.ld, 1)
    for i0 in starts:
        w = min(PANEL, n - i0)
        Xi = X.sub(i0, 0, w, nrhs)
        # Xi -= T[i, done] X[done]
        if lower and i0 > 0:
            _gemm(Xi, T.sub(i0, 0, w, i0), X.sub(0, 0, i0, nrhs), alpha=-1.0, beta=1.0, Cin=Xi)
        elif not lower and i0 + w < n:
            _gemm(Xi, T.sub(i0, i0 + w, w, n - i0 - w), X.sub(i0 + w, 0, n - i0 - w, nrhs),
                  alpha=-1.0, beta=1.0, Cin=Xi)
        Tii = T.sub(i0, i0, w, w)
        _lib.call("rs_trinv", Tii.ptr, rs_, cs_, None, w, int(lower), int(unit), inv.data_ptr(), PANEL,
                  _st())
        t2 = _device.Matrix(tmp, w, nrhs, max(nrhs, 1), False, X.kind)
        _gemm(t2, _device.Matrix(inv, w, w, PANEL, False, X.kind), Xi)
        _lib.call("rs_gather_rows", t2.ptr, t2.ld, None, w, nrhs, Xi.ptr, Xi.ld, _st())
    return X


def triangular_solve(t, b, side="left", uplo="lower", trans=False, unit_diagonal=False):
    """Triangular solve without forming the inverse of T (reference `dense.py:507-561`)."""
    tshape = _device.shape_of(t, "t")
    if tshape[0] != tshape[1]:
        raise DimensionError("triangular matrix must be square")
    if side not in ("left", "right"):
        raise ValueError(f"side must be 'left' or 'right', got {side!r}")
    if uplo not in ("lower", "upper"):
        raise ValueError(f"uplo must be 'lower' or 'upper', got {uplo!r}")
    T = _device.as_matrix(t, "t")
    kind = T.kind
    if not unit_diagonal and T.rows:
        d = T.tensor().diagonal()
        zero = torch.nonzero(d == 0.0)
        if zero.numel():
            raise SingularError(int(zero[0, 0]))
    if isinstance(b, torch.Tensor):
        bt = b.to(device=_device.device(), dtype=torch.float64)
    else:
        bt = torch.as_tensor(np.asarray(b, dtype=np.float64)).to(_device.device())
    squeeze = bt.dim() == 1
    if squeeze:
        bt = bt[:, None]
    lower = uplo == "lower"
    if side == "left":
        if T.cols != bt.shape[0]:
            raise DimensionError("dimension mismatch in triangular solve")
        M = T.T if trans else T
        low = lower != bool(trans)
        X = _trsm_left(M, _mat(bt.contiguous()), low, unit_diagonal).tensor()
    else:
        # X op(T) = B  <=>  op(T)^T X^T = B^T
        if T.rows != bt.shape[1]:
            raise DimensionError("dimension mismatch in triangular solve")
        M = T if trans else T.T
        low = lower == bool(trans)
        X = _trsm_left(M, _mat(bt.T.contiguous()), low, unit_diagonal).tensor().T
    if squeeze:
        X = X[:, 0]
    return _out(X.contiguous(), kind)


# ------------------------------------------------------------ small ops -----
def gemm(a, b, transpose_a=False, transpose_b=False):
    """``op(a) @ op(b)`` on the DMMA kernel (reference `dense.py:118-141`)."""
    sa = _device.shape_of(a, "a")
    sb = _device.shape_of(b, "b")
    ka = sa[0] if transpose_a else sa[1]
    kb = sb[1] if transpose_b else sb[0]
    if ka != kb:
        opa = (sa[1], sa[0]) if transpose_a else sa
        opb = (sb[1], sb[0]) if transpose_b else sb
        raise DimensionError(f"inner dimensions do not agree: {opa} x {opb}")
    A = _device.as_matrix(a, "a")
    B = _device.as_matrix(b, "b")
    if transpose_a:
        A = A.T
    if transpose_b:
        B = B.T
    C = _device.empty(A.rows, B.cols, A.kind)
    if A.rows and B.cols:
        if A.cols == 0:
            C.tensor().zero_()
        else:
            _gemm(C, A, B)
    return _out(C, A.kind)


def frobenius_norm(a):
    """``sqrt(sum a^2)`` with a deterministic device reduction (reference `dense.py:144-146`)."""
    if isinstance(a, torch.Tensor) and a.dim() == 1:
        a = a[:, None]
    elif not isinstance(a, torch.Tensor):
        arr = np.asarray(a, dtype=np.float64)
        a = arr.reshape(-1, 1) if arr.ndim <= 1 else arr.reshape(arr.shape[0], -1)
    X = _device.as_matrix(a)
    return math.sqrt(_sumsq(X)) if X.rows and X.cols else 0.0


def row_permute(a, perm):
    """``a[perm]`` (reference `dense.py:149-155`), via the device gather kernel."""
    m, n = _device.shape_of(a)
    p = np.asarray(perm.cpu() if isinstance(perm, torch.Tensor) else perm)
    if p.shape[0] != m:
        raise DimensionError("permutation length does not match row count")
    A = _device.as_matrix(a)
    out = _gather_rows(A, _ti(p))
    return _out(out, A.kind)


def invert_permutation(perm):
    """``inv[perm[i]] = i`` (reference `dense.py:158-163`)."""
    if isinstance(perm, torch.Tensor):
        p = perm.to(torch.int64)
        inv = torch.empty_like(p)
        inv[p] = torch.arange(p.numel(), dtype=torch.int64, device=p.device)
        return inv
    p = np.asarray(perm, dtype=np.intp)
    inv = np.empty_like(p)
    inv[p] = np.arange(p.shape[0], dtype=np.intp)
    return inv
