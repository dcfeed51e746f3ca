"""Two-sided ID and CUR on the B200 -- drop-in for `randskel.skeleton`
(`skeleton.py:565-647`) and `dense.pinv_apply` (`dense.py:166-182`).

  pinv_apply(a, b)            min-norm least squares, singular values below
                              1e-12 * sigma_max truncated (gelsd semantics),
                              by one-sided Jacobi SVD on the device
  two_sided_id(a, k, spec, rng)
  cur_decompose(a, k, spec, rng)

Skeleton gathers (`a[row_idx]`, `a[:, col_idx]`, `a[ix_(I, J)]`) run on the
gather kernel; column skeletons come from LUPP of ``a[row_idx].T`` on the
T-form engine; the 1-norm condition number of the skeleton submatrix is
estimated from its device LU with LAPACK dgecon's algorithm (Hager/Higham
dlacn2), as the reference's flag does.
"""

from dataclasses import dataclass

import numpy as np
import torch

from . import _device, _engine, _lib, dense
from .errors import DimensionError, RankDeficientError
from .skeleton import STATUS_ILL_CONDITIONED, STATUS_OK, SkeletonResult, rand_lupp

__all__ = ["CurFactors", "pinv_apply", "two_sided_id", "cur_decompose", "cur_decompose_adaptive"]

PINV_RCOND = 1e-12   # dense.py:49
COND_LIMIT = 1e14    # skeleton.py:72
JACOBI_TOL = 2.0 ** -52
JACOBI_SWEEPS = 40


@dataclass
class CurFactors:
    """C = a[:, col_idx], R = a[row_idx, :] implied (reference `skeleton.py:132-139`)."""

    row_idx: object
    col_idx: object
    u_mid: object
    status: str = STATUS_OK


def _st():
    return _device.stream_handle()


def _round_robin(q):
    """Circle-method schedule: q-1 rounds (q even) of q/2 disjoint pairs."""
    n = q + (q % 2)
    players = list(range(n))
    rounds = []
    for _ in range(n - 1):
        pr = []
        for i in range(n // 2):
            a, b = players[i], players[n - 1 - i]
            if a >= q or b >= q:
                a = b = -1
            pr.append((a, b))
        rounds.append(pr)
        players = [players[0]] + [players[-1]] + players[1:-1]
    return np.array(rounds, dtype=np.int32)  # (rounds, n/2, 2)


def _jacobi_svd_t(Xt):
    """One-sided Jacobi on Xt (q x p, rows = columns of X), in place.
    Returns Vt (q x q) with X V = Xt_final^T."""
    q, p = Xt.shape
    dev = Xt.device
    Vt = torch.eye(q, dtype=torch.float64, device=dev)
    if q <= 1:
        return Vt
    sched = torch.as_tensor(_round_robin(q)).to(dev)
    maxoff = torch.zeros(1, dtype=torch.int64, device=dev)
    bar = torch.zeros(1, dtype=torch.int32, device=dev)
    nrounds, npairs = sched.shape[0], sched.shape[1]
    for _ in range(JACOBI_SWEEPS):
        maxoff.zero_()
        # one cooperative launch per sweep; per-round launches if the pairs
        # do not fit co-resident (RS_ERR_CAPACITY)
        rc = _lib.load().rs_jacobi_sweep(Xt.data_ptr(), p, p, Vt.data_ptr(), q, q, sched.data_ptr(), nrounds,
                                         npairs, JACOBI_TOL, maxoff.data_ptr(), bar.data_ptr(), _st())
        if rc != 0:
            for r in range(nrounds):
                _lib.call("rs_jacobi_round", Xt.data_ptr(), p, p, Vt.data_ptr(), q, q,
                          sched[r].data_ptr(), npairs, JACOBI_TOL, maxoff.data_ptr(), _st())
        off = float(maxoff.view(torch.float64).item())
        if off <= JACOBI_TOL:
            break
    return Vt


def _pinv_apply_dev(A, B, b_planes=None):
    """x = A^+ B (A: Matrix p x q, B: Matrix p x r, any layouts) -> row-major tensor q x r.

    Tall A (p > 2q, q <= 1024) is first compressed to q x q: LUPP of A gives the
    interpolative form A = W A[I] (W = P [I; T], so sigma_min(W) >= 1 and W is
    well conditioned), CholeskyQR of W gives W = Q_W R_W, hence
    A = Q_W M with M = R_W A[I] (q x q) and A^+ B = M^+ (R_W^-T W^T B): the
    same singular values, so the rcond truncation is unchanged, and the
    Jacobi sweeps run on q x q instead of p x q.  Exactly rank-deficient or
    badly conditioned W falls back to Jacobi on A itself."""
    p, q = A.shape
    if p > 2 * q and 2 <= q <= 1024:
        x = _pinv_apply_compressed(A, B, b_planes)
        if x is not None:
            return x
    return _pinv_apply_jacobi(A, B)


def _pinv_apply_compressed(A, B, b_planes=None):
    p, q = A.shape
    r = B.cols
    dev = _device.device()
    Ar = A.row_major()
    st, W, fail = _engine.factor_sample(Ar, want_w=True)
    if fail is not None:
        return None
    Wm = dense._mat(W)                                   # p x q row-major
    A_I = _rows(Ar, st.perm[:q].clone())                 # q x q
    G = torch.empty((q, q), dtype=torch.float64, device=dev)
    dense._gemm(dense._mat(G), Wm.T, Wm)                 # W^T W = I + T^T T
    status = torch.empty(1, dtype=torch.int32, device=dev)
    _lib.call("rs_cholesky", G.data_ptr(), q, q, status.data_ptr(), _st())
    if int(status.item()) != 0:
        return None
    Rw = dense._mat(G)                                   # upper R_W, W = Q_W R_W
    M = torch.empty((q, q), dtype=torch.float64, device=dev)
    dense._gemm(dense._mat(M), Rw, A_I)                  # M = R_W A[I]
    # H = W^T B (q x r) without transposing a large column-major B
    if B.colmajor and b_planes is not None and b_planes.rows == r and b_planes.K == p:
        # B^T is the sketched matrix itself: H^T = B^T W on the int8 tensor cores,
        # from the digit planes the sketches already used (csrc/ozaki.cu)
        from . import _ozaki

        Ht = torch.empty((r, q), dtype=torch.float64, device=dev)
        _ozaki.sketch(b_planes, _ozaki.Planes.of_omega(W), Ht.data_ptr(), q)
        H = dense._mat(Ht).T.row_major()
    elif B.colmajor:
        Ht = torch.empty((r, q), dtype=torch.float64, device=dev)
        dense._gemm(dense._mat(Ht), B.T, Wm)             # H^T = B^T W
        H = dense._mat(Ht).T.row_major()
    else:
        Hr = torch.empty((q, r), dtype=torch.float64, device=dev)
        dense._gemm(dense._mat(Hr), Wm.T, B)
        H = dense._mat(Hr)
    H2 = dense._trsm_left(Rw.T, H, lower=True, unit=False)   # Q_W^T B = R_W^-T W^T B
    Mm = dense._mat(M)
    # gelsd truncates singular values below 1e-12 sigma_max.  When M is certainly far
    # from that (its 1-norm condition estimate < 1e10, so kappa_2 < sqrt(q) 1e10 <
    # 1e12), no value is truncated and M^+ = M^-1: solve by the device LU instead of
    # Jacobi sweeps.
    lu = _lu_factors(Mm)                                 # one LU for the estimate and the solve
    if lu is not None and _cond1(Mm, lu) < 1e10:
        return _lu_solve(Mm, H2, lu)
    return _pinv_apply_jacobi(Mm, H2)


def _lu_solve(M, B, lu=None):
    """X = M^-1 B for a square device Matrix M (LUPP + two blocked TRSMs); None when M is
    exactly singular."""
    if lu is None:
        lu = _lu_factors(M)
        if lu is None:
            return None
    perm, L, U = lu
    PB = _rows(B.row_major(), perm)                      # P B
    y = dense._trsm_left(dense._mat(L), PB, lower=True, unit=True)
    x = dense._trsm_left(dense._mat(U), y, lower=False, unit=False)
    return x.tensor()


def _pinv_apply_jacobi(A, B):
    """x = A^+ B by one-sided Jacobi on the columns of A: A V = U Sigma, then
    x = V diag(1/sigma^2) (A V)^T B with sigma <= rcond * sigma_max dropped."""
    p, q = A.shape
    r = B.cols
    dev = _device.device()
    Xt = _gather(A.T).tensor()          # q x p, rows = columns of A
    Vt = _jacobi_svd_t(Xt)
    sigma = torch.empty(max(q, 1), dtype=torch.float64, device=dev)
    _lib.call("rs_pinv_scale", Xt.data_ptr(), p, p, Vt.data_ptr(), q, q, PINV_RCOND, sigma.data_ptr(), _st())
    if B.colmajor:
        # Z^T = B^T (A V) with B^T row-major: no transpose of the (large) B
        XV = _gather(dense._mat(Xt).T)  # p x q row-major
        Zt = torch.empty((r, q), dtype=torch.float64, device=dev)
        dense._gemm(dense._mat(Zt), B.T, XV)
        Z = dense._mat(Zt).T            # q x r (column-major view)
    else:
        Zr = torch.empty((q, r), dtype=torch.float64, device=dev)
        dense._gemm(dense._mat(Zr), dense._mat(Xt), B)
        Z = dense._mat(Zr)
    x = torch.empty((q, r), dtype=torch.float64, device=dev)
    dense._gemm(dense._mat(x), dense._mat(Vt).T, Z)
    return x


def pinv_apply(a, b):
    """Minimum-norm least-squares solution of ``a @ x = b`` (reference `dense.py:166-182`)."""
    m, n = _device.shape_of(a, "a")
    if isinstance(b, torch.Tensor):
        bt = b.to(device=_device.device(), dtype=torch.float64)
    else:
        bt = torch.as_tensor(np.asarray(b, dtype=np.float64)).to(_device.device())
    if bt.dim() == 1:
        bt = bt[:, None]
    if m != bt.shape[0]:
        raise DimensionError(f"row counts do not agree: {(m, n)} vs {tuple(bt.shape)}")
    A = _device.as_matrix(a, "a")
    x = _pinv_apply_dev(A, dense._mat(bt.contiguous()))
    return dense._out(x, A.kind)


# ---------------------------------------------------------------- helpers ---
def _idx(x):
    if isinstance(x, torch.Tensor):
        return x.to(device=_device.device(), dtype=torch.int64)
    return torch.as_tensor(np.asarray(x, dtype=np.int64)).to(_device.device())


def _gather(A, ridx=None, cidx=None):
    """a[ridx][:, cidx] as a fresh row-major Matrix, any input layout (gather kernel)."""
    nr = A.rows if ridx is None else ridx.numel()
    nc = A.cols if cidx is None else cidx.numel()
    out = _device.empty(nr, nc, A.kind)
    rs_, cs_ = (1, A.ld) if A.colmajor else (A.ld, 1)
    _lib.call("rs_gather2d", A.ptr, rs_, cs_, ridx.data_ptr() if ridx is not None else None, nr,
              cidx.data_ptr() if cidx is not None else None, nc, out.ptr, out.ld, _st())
    return out


def _rows(A, idx):
    return _gather(A, ridx=idx)


def _cols(A, idx):
    return _gather(A, cidx=idx)


def _column_skeletons_from_rows(A, row_idx, k):
    """LUPP of a[row_idx].T (n x k) -> (col_idx, x) (reference `skeleton.py:565-571`)."""
    rows = _rows(A, row_idx)        # k x n
    y = rows.T.row_major()          # n x k
    st, w, fail = _engine.factor_sample(y, want_w=True)
    if fail is not None:
        raise RankDeficientError(fail)
    return st.perm[:k].clone(), w   # x = w.T


def _lu_factors(S):
    """Device LUPP of the k x k Matrix S: (perm, L, U) as device tensors, or None when S is
    exactly singular (dgetrf info > 0)."""
    k = S.rows
    A = S.row_major().copy()
    try:
        perm, _ = dense._lupp_device(A, allow_partial=False)
    except RankDeficientError:
        return None
    L, U = dense._split_lu(A, k)
    return perm, L.contiguous(), U.contiguous()


def _cond1(S, lu=None):
    """LAPACK-style 1-norm condition estimate of the k x k device Matrix S
    (`_condition_estimate_1norm`, skeleton.py:592-603: dgetrf + dgecon).

    The LU is the device LUPP (the same partial-pivoting rule as dgetrf; pass ``lu`` from
    `_lu_factors` to reuse one); ||S^-1||_1 is estimated by Hager/Higham's dlacn2
    iteration (at most five sign-vector steps plus the alternating-sign safeguard), every
    solve with the LU factors on the device TRSM, so the flag follows the reference's
    *estimate* rather than the exact condition number it bounds from below.  The host reads
    one small vector per iteration step.  Returns 1/rcond (inf for an exactly singular S or
    a zero S)."""
    k = S.rows
    dev = _device.device()
    out = torch.empty(1, dtype=torch.float64, device=dev)
    Sr = S.row_major()
    _lib.call("rs_norm1", Sr.ptr, Sr.ld, k, k, out.data_ptr(), _st())
    if lu is None:
        lu = _lu_factors(S)
    anorm = float(out.item())
    if anorm == 0.0 or lu is None:
        return np.inf  # zero S, or dgetrf info > 0
    _, L, U = lu
    st = _st()
    small = k <= 1024  # one-CTA column-oriented TRSV; larger k: the blocked device TRSM
    if small:
        Lt, Ut = L.t().contiguous(), U.t().contiguous()  # columns of L and U as rows
    else:
        Lm, Um = dense._mat(L), dense._mat(U)

    def solve(x, kase):
        """kase 1: x <- U^-1 L^-1 x ; kase 2: x <- L^-T U^-T x (dgecon's two dlatrs pairs)."""
        if not small:
            X = dense._mat(x.reshape(k, 1).contiguous())
            if kase == 1:
                y = dense._trsm_left(Lm, X, lower=True, unit=True)
                y = dense._trsm_left(Um, y, lower=False, unit=False)
            else:
                y = dense._trsm_left(Um.T, X, lower=True, unit=False)
                y = dense._trsm_left(Lm.T, y, lower=False, unit=True)
            return y.tensor().reshape(k)
        y = x.contiguous().clone()
        if kase == 1:
            _lib.call("rs_trsv_cols", Lt.data_ptr(), k, k, 1, 1, y.data_ptr(), st)   # L (unit lower)
            _lib.call("rs_trsv_cols", Ut.data_ptr(), k, k, 0, 0, y.data_ptr(), st)   # U (upper)
        else:
            _lib.call("rs_trsv_cols", U.data_ptr(), k, k, 1, 0, y.data_ptr(), st)    # U^T (lower)
            _lib.call("rs_trsv_cols", L.data_ptr(), k, k, 0, 1, y.data_ptr(), st)    # L^T (unit upper)
        return y

    def sgn(x):
        return torch.where(x >= 0, 1.0, -1.0).to(torch.float64)

    # dlacn2 (Higham 1988, LAPACK): reverse communication unrolled
    x = solve(torch.full((k,), 1.0 / k, dtype=torch.float64, device=dev), 1)
    if k == 1:
        est = float(x.abs()[0])
    else:
        est = float(x.abs().sum())
        isgn = sgn(x)
        x = solve(isgn, 2)
        j = int(torch.argmax(x.abs()))
        it = 2
        while True:
            e = torch.zeros(k, dtype=torch.float64, device=dev)
            e[j] = 1.0
            x = solve(e, 1)
            xs = sgn(x)
            est_new, same = torch.stack([x.abs().sum(), (xs == isgn).all().to(torch.float64)]).tolist()
            estold, est = est, est_new
            if same != 0.0 or est <= estold:
                break  # repeated sign vector / cycling
            isgn = xs
            x = solve(isgn, 2)
            ax = x.abs()
            jn = torch.argmax(ax)
            jlast = j
            jv, xl, xj = torch.stack([jn.to(torch.float64), x[jlast], ax[jn]]).tolist()
            j = int(jv)
            if xl != xj and it < 5:
                it += 1
                continue
            break
        alt = torch.arange(k, dtype=torch.float64, device=dev)
        alt = (1.0 + alt / (k - 1)) * torch.where(alt % 2 == 0, 1.0, -1.0).to(torch.float64)
        x = solve(alt, 1)
        temp = 2.0 * (float(x.abs().sum()) / (3 * k))
        if temp > est:
            est = temp
    if not np.isfinite(est):
        return np.inf
    if est == 0.0:
        return np.inf
    rcond = (1.0 / est) / anorm
    return np.inf if rcond == 0.0 else 1.0 / rcond


def two_sided_id(a, k, spec, rng):
    """Row skeletons by sketched LUPP, columns from the rows (reference `skeleton.py:606-625`)."""
    A = _device.as_matrix(a)          # one H2D of a host input, shared by every stage
    r = rand_lupp(A, k, spec, rng)
    ridx = _idx(r.row_idx)
    cidx, w = _column_skeletons_from_rows(A, ridx, k)
    S = _cols(_rows(A, ridx), cidx)
    status = STATUS_ILL_CONDITIONED if _cond1(S) > COND_LIMIT else STATUS_OK
    kind = A.kind
    x = _device.to_output(w, kind)
    return SkeletonResult(rank=k, row_idx=r.row_idx, col_idx=_device.to_host_index(cidx, kind),
                          w=r.w, x=x.T, status=status)


def cur_decompose(a, k, spec, rng):
    """CUR with skeletons from sketched LUPP and ``u_mid = C^+ a R^+``
    (reference `skeleton.py:628-647`)."""
    A = _device.as_matrix(a)          # one H2D of a host input, shared by every stage
    r = rand_lupp(A, k, spec, rng)
    ridx = _idx(r.row_idx)
    return _cur_from_rows(A, ridx, k, r.row_idx)


def _cur_from_rows(A, ridx, k, row_idx_out, planes=None):
    cidx, _ = _column_skeletons_from_rows(A, ridx, k)
    C = _cols(A, cidx)                   # m x k
    R = _rows(A, ridx)                   # k x n
    # a R^+ = pinv_apply(R^T, a^T)^T ;  u_mid = pinv_apply(C, a R^+)
    arp_t = _pinv_apply_dev(R.T, A.T, b_planes=planes)    # k x m  (= (a R^+)^T)
    u_mid = _pinv_apply_dev(C, dense._mat(arp_t).T)
    S = _cols(R, cidx)
    status = STATUS_ILL_CONDITIONED if _cond1(S) > COND_LIMIT else STATUS_OK
    kind = A.kind
    return CurFactors(row_idx=row_idx_out, col_idx=_device.to_host_index(cidx, kind),
                      u_mid=dense._out(u_mid, kind), status=status)


def cur_decompose_adaptive(a, b, tau, spec, rng, max_rank=None):
    """Adaptive CUR (BASELINE configs[2]): rows by `rand_lupp_adaptive` to
    tolerance tau, columns from the rows, linking matrix as `cur_decompose`.

    The reference has no adaptive CUR; this is the composition SURVEY.md 8c
    pins for it (`skeleton.py:391-460` then `skeleton.py:637-647` at the
    detected rank).  fp32 inputs are upcast to fp64 like the reference
    (`skeleton.py:200-204`).  Returns ``(CurFactors, SkeletonResult)``.
    """
    from . import _ozaki
    from .skeleton import _adaptive_device

    A = _device.as_matrix(a)
    # the digit planes of A serve both the sketches and the A R^+ product
    planes = _ozaki.Planes.of_matrix(A) if _ozaki.sketch_engine() == "ozaki" else None
    res = _adaptive_device(A, b, tau, spec, rng, max_rank=max_rank, planes=planes)
    ridx = _idx(res.row_idx)
    cur = _cur_from_rows(A, ridx, res.rank, res.row_idx, planes=planes)
    return cur, res
