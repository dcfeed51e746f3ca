"""T-form blocked LUPP engine (device-resident state of the skeleton loop).

State at rank k over m candidates (rows of the sketch):
  perm  (m,)        int64  -- perm[:k] skeletons in pivot order, perm[k:] the
                              remaining candidates in their *current position*
                              order (the reference's `state.perm`,
                              `skeleton.py:152-173`);
  T     (m-k) x k   fp64   -- T = L2 L1^{-1}, row i interpolates candidate
                              perm[k+i] from the skeletons.
The reference keeps (L1, L2, U1, ysofar) and re-solves L1 per block; the
T-form keeps only the interpolation block, so the per-block work is two
row-parallel DMMA GEMMs and there is no final triangular solve: W is ready
when the loop stops (north star: "without a second pass").

Per block of width w (`skeleton.py:439-454`):
  schur:  S = Y[perm[k:]] - T Y[perm[:k]],  e2 = ||S||^2   (rs_schur_block)
  panel:  S[pi] = L_hat U_hat with partial pivoting         (rs_panel_lupp)
  absorb: T' = [T[Q_hat] - W_hat T[P_hat], W_hat]          (rs_absorb_block)
All three are enqueued on the current torch stream; the host reads back
one scalar (e2) and one int (eliminated columns) per block.
"""

import numpy as np
import torch

from . import _device, _lib

MAX_BLOCK = 64


def _t_capacity(m, kcap):
    """max over k <= kcap of (m - k) * k (T is compact with ld = k)."""
    best = 0
    for k in {min(kcap, m // 2), min(kcap, (m + 1) // 2), kcap}:
        if 0 <= k <= m:
            best = max(best, (m - k) * k)
    return max(best, 1)


class TFormState:
    """Ping-pong device buffers for the T-form blocked LUPP over m candidates."""

    def __init__(self, m, kcap, bmax=MAX_BLOCK):
        if bmax > MAX_BLOCK:
            raise ValueError("block width above 64 is split by the caller")
        dev = _device.device()
        self.m = m
        self.k = 0
        cap = _t_capacity(m, kcap)
        self._T = [torch.empty(cap, dtype=torch.float64, device=dev) for _ in range(2)]
        self._perm = [torch.empty(max(m, 1), dtype=torch.int64, device=dev) for _ in range(2)]
        self._cur = 0
        # Schur block S (factored in place by the panel).  absorb_schur writes
        # the next block's S into the other buffer, so a rollback can still
        # re-absorb the previous block from its own factored S.
        self._S = [torch.empty(max(m * bmax, 1), dtype=torch.float64, device=dev)]
        self._scur = 0
        self.sub = torch.empty(max(m, 1), dtype=torch.int64, device=dev)
        self.ws = _device.workspace()
        self.stream = _device.stream_handle()
        _lib.call("rs_iota", self.perm.data_ptr(), m, self.stream)

    # -- views ---------------------------------------------------------------
    @property
    def S(self):
        return self._S[self._scur]

    def _s_next(self):
        if len(self._S) == 1:
            self._S.append(torch.empty_like(self._S[0]))
        return self._S[1 - self._scur]

    @property
    def perm(self):
        return self._perm[self._cur]

    @property
    def T(self):
        return self._T[self._cur]

    def t_matrix(self):
        """T as an (m-k) x k row-major tensor view."""
        k = self.k
        return self.T[: (self.m - k) * k].view(self.m - k, k)

    # -- block operations ------------------------------------------------------
    def schur(self, y_ptr, ldy, w, e2_out=None):
        """S = Y[perm[k:]] - T Y[perm[:k]] for the w-column block at y_ptr."""
        _lib.call(
            "rs_schur_block", self.m, self.k, w, y_ptr, ldy, self.perm.data_ptr(),
            self.T.data_ptr(), max(self.k, 1), self.S.data_ptr(), w,
            e2_out.data_ptr() if e2_out is not None else None, self.ws.data_ptr(), self.stream,
        )

    def panel(self, w, ncols_out):
        """LUPP of the (m-k) x w Schur block in S; ncols_out (device int32) gets
        the eliminated column count."""
        _lib.call(
            "rs_panel_lupp", self.S.data_ptr(), w, self.m - self.k, w, self.sub.data_ptr(),
            ncols_out.data_ptr(), self.ws.data_ptr(), self.stream,
        )

    def absorb(self, w, nc):
        """Fold the first nc factored columns of S into (T, perm)."""
        nxt = 1 - self._cur
        _lib.call(
            "rs_absorb_block", self.m, self.k, nc, self.S.data_ptr(), w, self.sub.data_ptr(),
            self.T.data_ptr(), max(self.k, 1), self._T[nxt].data_ptr(), self.perm.data_ptr(),
            self._perm[nxt].data_ptr(), self.ws.data_ptr(), self.stream,
        )
        self._prev = (self._cur, self.k, self._scur)
        self._cur = nxt
        self.k += nc

    def absorb_schur(self, w, nc, y_next_ptr, e2_out, ldy=64):
        """absorb(w, nc) fused with the Schur block of the next sketch block
        (m x 64 at y_next_ptr) into S, e2_out = ||S||^2 (rs_absorb_schur)."""
        nxt = 1 - self._cur
        s_next = self._s_next()
        _lib.call(
            "rs_absorb_schur", self.m, self.k, nc, self.S.data_ptr(), w, self.sub.data_ptr(),
            self.T.data_ptr(), max(self.k, 1), self._T[nxt].data_ptr(), self.perm.data_ptr(),
            self._perm[nxt].data_ptr(), y_next_ptr, ldy, s_next.data_ptr(),
            e2_out.data_ptr() if e2_out is not None else None, self.ws.data_ptr(), self.stream,
        )
        self._prev = (self._cur, self.k, self._scur)
        self._cur = nxt
        self._scur = 1 - self._scur
        self.k += nc

    def schur_next(self, y_ptr, ldy, e2_out, w=MAX_BLOCK):
        """After `absorb`: the next block's Schur block S' = Y'[perm'[k:]] -
        T' Y'[perm'[:k]] into the other S buffer (the absorbed block's factored
        S stays intact for a rollback) -- the second half of `absorb_schur`."""
        s_next = self._s_next()
        _lib.call(
            "rs_schur_block", self.m, self.k, w, y_ptr, ldy, self.perm.data_ptr(), self.T.data_ptr(),
            max(self.k, 1), s_next.data_ptr(), w, e2_out.data_ptr() if e2_out is not None else None,
            self.ws.data_ptr(), self.stream,
        )
        self._scur = 1 - self._scur  # (_prev, set by absorb, keeps the factored S)

    def rollback(self):
        """Undo the last absorb (its inputs are intact in the other buffers):
        used when a speculative absorb assumed a full-width elimination."""
        self._cur, self.k, self._scur = self._prev

    def interpolation(self, out=None):
        """Dense W (m x k) with W[perm[:k]] = I, W[perm[k:]] = T."""
        k = self.k
        if out is None:
            out = torch.empty((self.m, k), dtype=torch.float64, device=self.T.device)
        _lib.call("rs_scatter_interp", self.T.data_ptr(), max(k, 1), self.perm.data_ptr(),
                  self.m, k, out.data_ptr(), max(k, 1), self.stream)
        return out


def factor_sample(y, want_w=True):
    """One-shot LUPP of a device sketch ``y`` (m x ell row-major Matrix) in
    64-column blocks through the T-form engine.  Mirrors `lupp(y)` followed
    by `_w_from_lu` (`skeleton.py:185-189`).

    Returns ``(state, w, fail_step)``: fail_step is None or the 0-based
    elimination step of the first exactly-zero pivot column
    (`RankDeficientError(step)`, `dense.py:195-198`).
    """
    m, ell = y.shape
    st = TFormState(m, ell, min(MAX_BLOCK, max(ell, 1)))
    nblk = (ell + MAX_BLOCK - 1) // MAX_BLOCK
    ncols = torch.empty(max(nblk, 1), dtype=torch.int32, device=y.t.device)
    for bi in range(nblk):
        j0 = bi * MAX_BLOCK
        w = min(MAX_BLOCK, ell - j0)
        st.schur(y.ptr + 8 * j0, y.ld, w)
        st.panel(w, ncols[bi:])
        st.absorb(w, w)
    nc = ncols.cpu().numpy() if nblk else np.zeros(0, np.int32)
    fail = None
    for bi in range(nblk):
        w = min(MAX_BLOCK, ell - bi * MAX_BLOCK)
        if nc[bi] < w:
            fail = bi * MAX_BLOCK + int(nc[bi])
            break
    w_mat = st.interpolation() if (want_w and fail is None) else None
    return st, w_mat, fail
