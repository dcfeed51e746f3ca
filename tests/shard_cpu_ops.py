"""CPU test double of `sharded.DeviceShardOps` (test infrastructure only).

Implements the same per-rank primitives with numpy / torch-CPU tensors so the
sharded loop's host logic -- ownership maps, exchanges over torch.distributed
(gloo), stop rule -- runs world_size > 1 on a machine without a GPU.  The
panel is the oracle's LUPP (`oracle/randskel_oracle.py:lupp_inplace`, the
restatement of `dense.py:185-233`) and Omega the oracle's numpy draw.
"""

import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle"))
import randskel_oracle as orc  # noqa: E402


def _np(t):
    return t.numpy()


class CpuShardOps:
    def __init__(self, a_local, seed, stream=0):
        self.a = np.ascontiguousarray(a_local, dtype=np.float64)
        self.dev = torch.device("cpu")
        self.seed, self.stream = seed, stream

    def f64(self, n):
        return torch.full((max(int(n), 1),), np.nan, dtype=torch.float64)

    def i64(self, n):
        return torch.full((max(int(n), 1),), -7, dtype=torch.int64)

    def i32(self, n):
        return torch.zeros(max(int(n), 1), dtype=torch.int32)

    def omega(self, rng, t, b):
        return orc.gaussian(self.seed, orc.child_stream(self.stream, t), self.a.shape[1], b)

    def sketch(self, om, b, out):
        m, n = self.a.shape
        _np(out)[: m * b] = (self.a @ om).ravel()

    def sketch_structured(self, spec, rng, t, b, out):
        m, n = self.a.shape
        st = orc.child_stream(self.stream, t)
        if spec.kind == "sparsesign":
            idx, sg, sc = orc.sparse_sign_operator(self.seed, st, n, b, min(spec.zeta, b))
            y = orc.sparse_sign_apply(self.a, idx, sg, sc, b)
        else:
            y = self.a @ orc.srtt_dense(self.seed, st, n, b)
        _np(out)[: m * b] = y.ravel()

    def iota(self, p, n):
        _np(p)[:n] = np.arange(n)

    def gather_rows(self, src, lds, idx, n, cols, dst, ldd):
        s, d, ix = _np(src), _np(dst), _np(idx)
        for i in range(n):
            r = int(ix[i])
            d[i * ldd: i * ldd + cols] = 0.0 if r < 0 else s[r * lds: r * lds + cols]

    def scatter_rows(self, src, lds, idx, n, cols, dst, ldd):
        s, d, ix = _np(src), _np(dst), _np(idx)
        for i in range(n):
            r = int(ix[i])
            if r >= 0:
                d[r * ldd: r * ldd + cols] = s[i * lds: i * lds + cols]

    def schur(self, r, k, b, Tg, Ytop, Y, loc, out, ldy=None):
        ldy = b if ldy is None else ldy
        rows = _np(loc)[:r].astype(np.int64)
        y = _np(Y)[rows[:, None] * ldy + np.arange(b)[None, :]]
        if k > 0:
            y = y - _np(Tg)[: r * k].reshape(r, k) @ _np(Ytop)[: k * b].reshape(k, b)
        _np(out)[: r * b] = y.ravel()

    def sumsq(self, X, R, w, out):
        x = _np(X)[: R * w]
        _np(out)[0] = float(x @ x)

    def panel(self, S, R, w, sub, ncols):
        s = _np(S)[: R * w].reshape(R, w)
        A = np.array(s, order="F")
        perm, nc = orc.lupp_inplace(A, allow_partial=True)
        s[perm] = A
        _np(sub)[:R] = perm
        _np(ncols)[0] = nc

    def perm_update(self, perm, perm_new, m, k, sub):
        p, q, s = _np(perm), _np(perm_new), _np(sub)
        q[:k] = p[:k]
        q[k:m] = p[k + s[: m - k]]

    def maps(self, perm, m, k, lo, hi, lrow_old, sub, k_old, nc, lrow, loc, spos, src_row, wsrc, tp_src,
             ytop_src, count, pad_to=0):
        p = _np(perm)[:m]
        own = (p >= lo) & (p < hi)
        ys = _np(ytop_src)
        ys[:k] = np.where(own[:k], p[:k] - lo, -1)
        lr = _np(lrow)
        lr[:m] = -1
        pos = np.flatnonzero(own[k:]) + k
        r = len(pos)
        lr[pos] = np.arange(r)
        _np(loc)[:r] = p[pos] - lo
        _np(spos)[:r] = pos - k
        if sub is not None:
            s, lo_old = _np(sub), _np(lrow_old)
            j = s[pos - k_old]
            _np(src_row)[:r] = lo_old[k_old + j]
            _np(wsrc)[:r] = j
            _np(tp_src)[:nc] = lo_old[k_old + s[:nc]]
        if pad_to > r:
            _np(loc)[r:pad_to] = 0
            _np(spos)[r:pad_to] = -1
            if sub is not None:
                _np(src_row)[r:pad_to] = 0
                _np(wsrc)[r:pad_to] = 0
        _np(count)[0] = r

    def max_count(self, perm, m, k, bounds, world, out):
        p, bnd = _np(perm)[k:m], _np(bounds)[: world + 1]
        _np(out)[0] = max(int(((p >= bnd[g]) & (p < bnd[g + 1])).sum()) for g in range(world))

    def what(self, S, lds, sub, nc, wsrc, r, linv, out, ldo):
        s = _np(S)
        rows = np.stack([s[int(i) * lds: int(i) * lds + nc] for i in _np(sub)[:nc]])
        L1 = np.tril(rows, -1) + np.eye(nc)
        li = np.linalg.inv(L1)
        o = _np(out)
        for i in range(r):
            j = int(_np(wsrc)[i])
            o[i * ldo: i * ldo + nc] = s[j * lds: j * lds + nc] @ li

    def t_update(self, r, k, nc, Tn, ldn, TP, iota, Tg, src_row):
        tn, tp, tg = _np(Tn), _np(TP)[: nc * k].reshape(nc, k), _np(Tg)
        for i in range(r):
            j = int(_np(src_row)[i])
            w = tn[i * ldn + k: i * ldn + k + nc]
            tn[i * ldn: i * ldn + k] = tg[j * k: j * k + k] - w @ tp

    def scatter_interp_local(self, Tg, k, perm, loc, r, lo, hi, W):
        mg = hi - lo
        w = _np(W)[: mg * k].reshape(mg, k)
        w[:] = 0.0
        p = _np(perm)
        for i in range(k):
            if lo <= p[i] < hi:
                w[p[i] - lo, i] = 1.0
        tg = _np(Tg)
        for i in range(r):
            w[int(_np(loc)[i])] = tg[i * k: i * k + k]

    def read(self, *xs):
        return [x.item() for x in xs]

    def output(self, row_idx, w):
        return row_idx.numpy(), w.numpy()
