"""Column-sharded adaptive skeleton loop over ranks.

The reference is single-process; its north-star multi-GPU form is the
column ID of an A that is column-sharded across the GPUs of one box: rank g
holds the contiguous candidate rows ``a[lo:hi]`` of ``a = A.T`` (so A's
columns J_g) and the loop of `rand_lupp_adaptive` (`skeleton.py:391-460`)
runs with

  * the sketch ``Y_g = a[lo:hi] @ Omega_t`` fully local -- every rank draws
    the same Omega_t = rng.child(t) on its own device (no broadcast);
  * ONE exchange of the pivot candidates per block: the Schur block
    ``S = Y[perm[k:]] - T Y[perm[:k]]`` is formed row-parallel (each rank its
    own remaining candidates, against the all-reduced skeleton rows Y_top)
    and all-reduced into position order, so every rank runs the SAME exact
    partial-pivoting panel on the same S (no tournament pivoting; pivots,
    e_schur and the stop decision are identical on all ranks);
  * the pivots' interpolation rows T[P_hat] all-reduced once per block for
    the rank-nc update of the local rows T_g.

The all-reduces carry one nonzero contribution per element (owners write,
the others write zeros), so they are exact: the result does not depend on
the reduction order or on the world size.  The position order ``perm`` is
replicated; T_g stays local and compact (rows = the rank's remaining
candidates in position order).  At the end ``row_idx = perm[:k]`` is
global and W stays row-sharded: the rank gets ``W[lo:hi]``.

The per-rank arithmetic is behind a small ops object: `DeviceShardOps`
(librskel.so kernels, the product path) or a test double.
"""

import math

import torch
import torch.distributed as dist

from . import _device, _lib, _ozaki
from .errors import DimensionError, RankDeficientError
from .skeleton import (
    STATUS_NOT_CONVERGED,
    STATUS_OK,
    STATUS_RANK_EXHAUSTED,
    ErrorTrace,
    SkeletonResult,
    TraceRecord,
)

__all__ = ["DeviceShardOps", "rand_lupp_adaptive_sharded", "shard_bounds"]

MAX_BLOCK = 64


def shard_bounds(m, world, rank):
    """Contiguous near-equal split of m candidates: rank -> [lo, hi)."""
    base, extra = divmod(m, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


class DeviceShardOps:
    """Per-rank primitives on librskel.so (all on the current stream)."""

    def __init__(self, a_local):
        self.a = a_local
        self.dev = _device.device()
        self.ws = _device.workspace()
        self.st = _device.stream_handle()
        self.host_rng = _device.host_rng()
        self.rng_status = torch.zeros(4096, dtype=torch.int32, device=self.dev)
        # tensor-core sketch: the local candidates' digit planes, cut once
        self.ap = _ozaki.Planes.of_matrix(a_local) if _ozaki.sketch_engine() == "ozaki" else None
        self.bp = None
        self.side = None  # look-ahead sketch stream (created on first use)

    def f64(self, n):
        return torch.empty(max(int(n), 1), dtype=torch.float64, device=self.dev)

    def i64(self, n):
        return torch.empty(max(int(n), 1), dtype=torch.int64, device=self.dev)

    def i32(self, n):
        return torch.empty(max(int(n), 1), dtype=torch.int32, device=self.dev)

    def omega(self, rng, t, b):
        """Omega_t = rng.child(t) Gaussian block (n x b), drawn on this device
        without a host sync (statuses checked once at the end, `rng_ok`)."""
        n = self.a.shape[1]
        if self.host_rng:
            return torch.as_tensor(_device.host_gaussian(rng.child(t), n, b)).to(self.dev)
        slot = t % self.rng_status.numel()
        return _device.gaussian(rng.child(t), n, b, status=self.rng_status[slot:slot + 1])

    def rng_ok(self):
        """True if every device draw was resolved (else rerun with host draws)."""
        if self.host_rng or not bool(self.rng_status.any()):
            return True
        self.host_rng = True
        self.rng_status.zero_()
        return False

    def sketch(self, om, b, out, ws=None):
        m, n = self.a.shape
        ws = self.ws if ws is None else ws
        st = _device.stream_handle()
        if self.ap is not None:
            if self.bp is None:
                self.bp = _ozaki.Planes(b, n, _ozaki.OMEGA_PLANES, 64, self.dev)
            _ozaki.Planes.of_omega(om, out=self.bp, ws=ws)
            return _ozaki.sketch(self.ap, self.bp, out.data_ptr(), b, ws=ws)
        _lib.call("rs_sketch_gemm", m, n, b, self.a.ptr, self.a.ld, int(self.a.colmajor), om.data_ptr(), b,
                  out.data_ptr(), b, ws.data_ptr(), st)

    def sketch_structured(self, spec, rng, t, b, out):
        """Block t of an SRTT / sparse-sign embedding on the local rows: the
        reference's operator from rng.child(t); sparse sign as the SpMM (bitwise
        the reference's rows), SRTT dense through the sketch engine."""
        from .lu_state import _block_spec
        from .sketching import make_sketch

        m, n = self.a.shape
        op = make_sketch(_block_spec(spec, n, b), rng.child(t))
        if spec.kind == "sparsesign":
            _device.sparse_sign_apply(self.a, op.idx, op.signs, op.ell, op.scale, out=out[: m * b].view(m, b))
        else:
            self.sketch(op.device_dense(), b, out)

    def sketch_async(self, rng, t, b, out, prof=None):
        """Omega_t draw + sketch on a side stream (own workspace), so they
        overlap the current block's exchanges and panel; `wait_sketch` joins."""
        if self.side is None:
            self.side = torch.cuda.Stream(device=self.dev)
            self.ws_side = _device.workspace(slot=1)
        self.side.wait_stream(torch.cuda.current_stream(self.dev))
        with torch.cuda.stream(self.side):
            om = self.omega(rng, t, b)
            tok = prof.start("sketch_gemm") if prof is not None else None
            self.sketch(om, b, out, ws=self.ws_side)
            if tok is not None:
                prof.stop(tok)

    def wait_sketch(self):
        if self.side is not None:
            torch.cuda.current_stream(self.dev).wait_stream(self.side)

    def max_count(self, perm, m, k, bounds, world, out):
        _lib.call("rs_shard_max_count", perm.data_ptr(), m, k, bounds.data_ptr(), world, out.data_ptr(), self.st)

    def iota(self, p, n):
        _lib.call("rs_iota", p.data_ptr(), n, self.st)

    def gather_rows(self, src, lds, idx, n, cols, dst, ldd):
        _lib.call("rs_gather_rows", src.data_ptr(), lds, idx.data_ptr(), n, cols, dst.data_ptr(), ldd, self.st)

    def scatter_rows(self, src, lds, idx, n, cols, dst, ldd):
        _lib.call("rs_scatter_rows", src.data_ptr(), lds, idx.data_ptr(), n, cols, dst.data_ptr(), ldd, self.st)

    def schur(self, r, k, b, Tg, Ytop, Y, loc, out, ldy=None):
        """out (r x b) = Y[loc] - Tg (r x k) @ Ytop (k x b); Y rows ldy apart (default b)."""
        ldy = b if ldy is None else ldy
        if k == 0:
            return self.gather_rows(Y, ldy, loc, r, b, out, b)
        _lib.call("rs_dgemm", r, b, k, -1.0, Tg.data_ptr(), k, 0, None, Ytop.data_ptr(), b, None, 1.0,
                  Y.data_ptr(), ldy, loc.data_ptr(), out.data_ptr(), b, self.ws.data_ptr(), self.st)

    def sumsq(self, X, R, w, out):
        _lib.call("rs_sumsq", X.data_ptr(), w, R, w, out.data_ptr(), self.ws.data_ptr(), self.st)

    def panel(self, S, R, w, sub, ncols):
        _lib.call("rs_panel_lupp", S.data_ptr(), w, R, w, sub.data_ptr(), ncols.data_ptr(), self.ws.data_ptr(),
                  self.st)

    def perm_update(self, perm, perm_new, m, k, sub):
        _lib.call("rs_perm_update", perm.data_ptr(), perm_new.data_ptr(), m, k, sub.data_ptr(), self.st)

    def maps(self, perm, m, k, lo, hi, lrow_old, sub, k_old, nc, lrow, loc, spos, src_row, wsrc, tp_src,
             ytop_src, count, pad_to=0):
        p = (lambda x: x.data_ptr() if x is not None else None)
        _lib.call("rs_shard_maps", perm.data_ptr(), m, k, lo, hi, p(lrow_old), p(sub), k_old, nc, lrow.data_ptr(),
                  loc.data_ptr(), spos.data_ptr(), p(src_row), p(wsrc), p(tp_src), ytop_src.data_ptr(),
                  count.data_ptr(), pad_to, self.st)

    def what(self, S, lds, sub, nc, wsrc, r, linv, out, ldo):
        """out[i, :nc] = S[wsrc[i]] L1^{-1}, L1 = unit lower part of rows S[sub[:nc]]
        (the same substitution kernel as the single-GPU absorb)."""
        if r > 0:
            _lib.call("rs_what", S.data_ptr(), lds, sub.data_ptr(), nc, wsrc.data_ptr(), r, out.data_ptr(), ldo,
                      self.st)

    def t_update(self, r, k, nc, Tn, ldn, TP, iota, Tg, src_row):
        """Tn[:, :k] = Tg[src_row] - Tn[:, k:k+nc] @ TP (nc x k)."""
        if r == 0:
            return
        _lib.call("rs_rank_update", r, k, nc, Tn.data_ptr() + 8 * k, ldn, TP.data_ptr(), k, iota.data_ptr(),
                  Tg.data_ptr(), k, src_row.data_ptr(), Tn.data_ptr(), ldn, self.st)

    def scatter_interp_local(self, Tg, k, perm, loc, r, lo, hi, W):
        _lib.call("rs_scatter_interp_local", Tg.data_ptr(), max(k, 1), perm.data_ptr(), k, loc.data_ptr(), r,
                  lo, hi, W.data_ptr(), max(k, 1), self.st)

    def read(self, *xs):
        """Host values of small device scalars (one sync)."""
        return [x.item() for x in xs]

    def output(self, row_idx, w):
        """Results in the caller's container (numpy in -> numpy out, ...)."""
        return _device.to_host_index(row_idx, self.a.kind), _device.to_output(w, self.a.kind)


def _world(group):
    """(world size, rank); a process without a process group is rank 0 of 1."""
    if not dist.is_available() or not dist.is_initialized():
        return 1, 0
    return dist.get_world_size(group), dist.get_rank(group)


def _allreduce(x, group):
    if _world(group)[0] > 1:
        dist.all_reduce(x, op=dist.ReduceOp.SUM, group=group)


def _row_counts(m_local, group, dev):
    world = _world(group)[0]
    if world == 1:
        return [m_local]
    mine = torch.tensor([m_local], dtype=torch.int64, device=dev)
    allc = [torch.zeros(1, dtype=torch.int64, device=dev) for _ in range(world)]
    dist.all_gather(allc, mine, group=group)
    return [int(c.item()) for c in allc]


def rand_lupp_adaptive_sharded(a_local, b, tau, spec, rng, max_rank=None, group=None, ops=None):
    """`rand_lupp_adaptive` over ranks that each hold a contiguous block of
    the candidate rows (rank order = row order).  Same stopping rule, trace
    and statuses; returns a SkeletonResult whose ``row_idx``/``rank``/
    ``trace``/``status`` are global (identical on every rank) and whose ``w``
    holds this rank's rows of W.  Any block width: b <= 64 is one panel per block
    (pipelined), b > 64 is factored as 64-column panels (`_run_wide`).
    """
    if ops is None:
        a_local = _device.as_matrix(a_local)
        ops = DeviceShardOps(a_local)
        if ops.ap is not None:  # the digit planes drop NaN/inf: check the slicer's flag on every rank
            bad = ops.ap.nonfinite.clone()
            if _world(group)[0] > 1:
                dist.all_reduce(bad, op=dist.ReduceOp.MAX, group=group)
            if int(bad.item()):
                raise ValueError("matrix contains non-finite entries")
    m_loc, n = ops.a.shape
    counts = _row_counts(m_loc, group, ops.dev)
    rank = _world(group)[1]
    lo = sum(counts[:rank])
    hi = lo + m_loc
    m = sum(counts)
    if tau <= 0:
        raise ValueError(f"tau must be positive, got {tau}")
    if not 1 <= b <= min(m, n):
        raise DimensionError(f"block size must be in [1, {min(m, n)}], got {b}")
    if max_rank is None:
        max_rank = max(b, min(m, n) - b)
    max_rank = min(max_rank, min(m, n))
    res = _ShardedLoop(ops, group, m, n, lo, hi, b, tau, rng, max_rank, counts, spec).run()
    ok = torch.tensor([1 if (not hasattr(ops, "rng_ok") or ops.rng_ok()) else 0], dtype=torch.int32,
                      device=ops.dev)
    if _world(group)[0] > 1:
        dist.all_reduce(ok, op=dist.ReduceOp.MIN, group=group)
    if int(ok.item()) == 0:  # a draw the device resolver could not place (never observed): host draws
        if hasattr(ops, "host_rng"):
            ops.host_rng = True
        res = _ShardedLoop(ops, group, m, n, lo, hi, b, tau, rng, max_rank, counts, spec).run()
    return res


class _ShardedLoop:
    """One host readback per block, as the single-GPU driver: the absorb of
    block t is enqueued assuming a full-width elimination (nc = b) and sized
    by the previous exact local row count (an upper bound; padded map entries
    are inert); block t+1's sketch and Schur exchange follow at once, and one
    readback returns (e2 of t+1, eliminated columns of t, new row count).  A
    short block (an exactly zero pivot) is re-absorbed from its own factored
    Schur block, kept in the other S buffer."""

    def __init__(self, ops, group, m, n, lo, hi, b, tau, rng, max_rank, counts=None, spec=None):
        self.ops, self.group = ops, group
        # SRTT / sparse sign: the reference's per-block operator (`skeleton.py:286-295`),
        # the same on every rank (drawn from rng.child(t)), applied to the local rows
        self.spec = spec if spec is not None and spec.kind != "gaussian" else None
        self.m, self.n, self.lo, self.hi = m, n, lo, hi
        self.b, self.tau, self.rng, self.max_rank = b, tau, rng, max_rank
        mg = hi - lo
        counts = counts or [mg]
        self.world = len(counts)
        mg_max = max(counts)  # map arrays and Schur rows sized for the largest shard (all-gather padding)
        kcap = min(max_rank + b, m)
        o = ops
        self.perm = [o.i64(m), o.i64(m)]
        self.lrow = [o.i64(m), o.i64(m)]
        self.loc, self.spos, self.src_row, self.wsrc = o.i64(mg_max), o.i64(mg_max), o.i64(mg_max), o.i64(mg_max)
        self.tp_src, self.ytop_src = o.i64(b), o.i64(kcap)
        # [ncols of the last panel, local row count after the last maps, max count over ranks]
        self.meta = o.i32(3)
        self.pmax = mg_max   # all-gather rows per rank (an upper bound of every rank's count)
        if self.world > 1:
            bnd = [0]
            for c in counts:
                bnd.append(bnd[-1] + c)
            self.bounds = o.i64(self.world + 1)
            self.bounds[: self.world + 1] = torch.tensor(bnd, dtype=torch.int64)
            self.recv = o.f64(self.world * mg_max * b)
            self.recv_pos = o.i64(self.world * mg_max)
        self.sub = o.i64(m)
        self.iota_b = o.i64(b)
        o.iota(self.iota_b, b)
        self.Ys = [o.f64(mg * b), o.f64(mg * b)]  # sketch of block t and the look-ahead t+1
        self.Ytop = o.f64(kcap * b)
        self.Sg = o.f64(mg_max * b)
        self.S = [o.f64(m * b), o.f64(m * b)]
        self.scur = 0
        self.TP = o.f64(b * kcap)
        self.linv = o.f64(MAX_BLOCK * MAX_BLOCK)
        self.e2 = o.f64(1)
        # T rows are written up to the row-count bound (<= min(mg, m - k_old)) at ld k_new
        pts = {kcap, min(kcap, max(0, m - mg + b)), min(kcap, (m + b) // 2), min(kcap, (m + b + 1) // 2)}
        cap = max(1, max(min(mg, m - kk + b) * kk for kk in pts))
        self.T = [o.f64(cap), o.f64(cap)]
        self.cur = 0
        self.k = 0
        self.r = mg  # upper bound of the local row count (exact after each readback)

    def _schur(self, Y, j0=0, w=None):
        """Schur block of columns [j0, j0 + w) of the block sketch Y (rows b
        apart) into S (R x w, position order) and its squared norm into e2."""
        o, b, k = self.ops, self.b, self.k
        w = b if w is None else w
        Yj = Y[j0:] if j0 else Y
        Tg = self.T[self.cur]
        if k > 0:
            o.gather_rows(Yj, b, self.ytop_src, k, w, self.Ytop, w)
            _allreduce(self.Ytop[: k * w], self.group)
        if w == b:
            o.schur(self.r, k, w, Tg, self.Ytop, Yj, self.loc, self.Sg)
        else:
            o.schur(self.r, k, w, Tg, self.Ytop, Yj, self.loc, self.Sg, ldy=b)
        R = self.m - k
        S = self.S[self.scur][: R * w]
        if self.world == 1:
            o.scatter_rows(self.Sg, w, self.spos, self.r, w, S, w)
        else:
            # the one exchange of pivot candidates: every rank's Schur rows and their
            # positions (padded to P rows, padding at position -1) all-gathered, then
            # scattered into position order -- R (w + 1) words per rank received
            P = self.pmax
            recv, rpos = self.recv[: self.world * P * w], self.recv_pos[: self.world * P]
            dist.all_gather_into_tensor(recv, self.Sg[: P * w], group=self.group)
            dist.all_gather_into_tensor(rpos, self.spos[:P], group=self.group)
            o.scatter_rows(recv, w, rpos, self.world * P, w, S, w)
        o.sumsq(S, R, w, self.e2)

    def _absorb(self, nc, w=None):
        """Fold nc factored columns of the current S (R x w, default w = b) into
        (T, perm); launches sized by the row-count bound self.r."""
        o, m = self.ops, self.m
        b = self.b if w is None else w
        k_old, cur, S = self.k, self.cur, self.S[self.scur]
        k_new = k_old + nc
        nxt = 1 - cur
        rb = self.r
        o.perm_update(self.perm[cur], self.perm[nxt], m, k_old, self.sub)
        o.maps(self.perm[nxt], m, k_new, self.lo, self.hi, self.lrow[cur], self.sub, k_old, nc, self.lrow[nxt],
               self.loc, self.spos, self.src_row, self.wsrc, self.tp_src, self.ytop_src, self.meta[1:2],
               max(rb, self.pmax if self.world > 1 else 0))
        if self.world > 1:
            o.max_count(self.perm[nxt], m, k_new, self.bounds, self.world, self.meta[2:3])
        Tg, Tn = self.T[cur], self.T[nxt]
        if k_old > 0 and nc > 0:
            o.gather_rows(Tg, k_old, self.tp_src, nc, k_old, self.TP, k_old)
            _allreduce(self.TP[: nc * k_old], self.group)
        if nc > 0:
            o.what(S, b, self.sub, nc, self.wsrc, rb, self.linv, Tn[k_old:], k_new)
            if k_old > 0:
                o.t_update(rb, k_old, nc, Tn, k_new, self.TP, self.iota_b, Tg, self.src_row)
        self._prev = (cur, k_old)
        self.cur, self.k = nxt, k_new

    def _sketch_block(self, t, out):
        o, b = self.ops, self.b
        if self.spec is not None:
            o.sketch_structured(self.spec, self.rng, t, b, out)
        else:
            o.sketch(o.omega(self.rng, t, b), b, out)

    def _run_wide(self):
        """b > 64 (the paper's b = 128): each block is factored as 64-column
        panels, the single-GPU wide path (`_absorb_block`, the blocked
        `_lupp_partial` of `skeleton.py:318-351`): e_schur sums the sub-blocks'
        squared norms against the state before the block; then each sub-block's
        Schur rows are formed against the state that already holds the earlier
        sub-blocks, exchanged, factored and absorbed.  Synchronous per panel."""
        o, b, m, tau = self.ops, self.b, self.m, self.tau
        trace = ErrorTrace()
        status = STATUS_NOT_CONVERGED
        t = 0
        while True:
            Y = self.Ys[t % 2]
            self._sketch_block(t, Y)
            e2 = 0.0
            for j0 in range(0, b, MAX_BLOCK):
                self._schur(Y, j0, min(MAX_BLOCK, b - j0))
                e2 += float(o.read(self.e2)[0])
            if t > 0:
                e_schur = math.sqrt(e2) if e2 >= 0 else float("nan")
                trace.append(TraceRecord(k=self.k, e_schur=e_schur))
                if e_schur <= tau:
                    status = STATUS_OK
                    break
                if self.k + b > self.max_rank:
                    break
            if not math.isfinite(e2):
                raise ValueError("matrix contains non-finite entries")
            done = 0
            for j0 in range(0, b, MAX_BLOCK):
                w = min(MAX_BLOCK, b - j0)
                self._schur(Y, j0, w)
                o.panel(self.S[self.scur], m - self.k, w, self.sub, self.meta[0:1])
                (nc,) = o.read(self.meta[0:1])
                self._absorb(nc, w)
                if self.world > 1:
                    self.r, self.pmax = o.read(self.meta[1:2], self.meta[2:3])
                else:
                    (self.r,) = o.read(self.meta[1:2])
                done += nc
                if nc < w:
                    break
            if done < b:
                if t == 0:
                    raise RankDeficientError(done)
                status = STATUS_RANK_EXHAUSTED
                break
            t += 1
        return trace, status

    def run(self):
        o, b, m, tau = self.ops, self.b, self.m, self.tau
        o.iota(self.perm[0], m)
        o.maps(self.perm[0], m, 0, self.lo, self.hi, None, None, 0, 0, self.lrow[0], self.loc, self.spos, None,
               None, None, self.ytop_src, self.meta[1:2], self.pmax if self.world > 1 else 0)
        if b > MAX_BLOCK:
            trace, status = self._run_wide()
            return self._result(trace, status)
        trace = ErrorTrace()
        status = STATUS_NOT_CONVERGED
        from . import skeleton

        prof = skeleton._PHASE_TIMER or skeleton._NullTimer()
        pending = False  # speculative full-width absorb awaiting its ncols
        sketched = set()

        ahead_ok = hasattr(o, "sketch_async") and self.spec is None

        def sketch(tt, ahead=False):
            if tt in sketched:
                if ahead_ok:
                    o.wait_sketch()  # the look-ahead sketch of tt is done on the compute stream's clock
                return
            sketched.add(tt)
            if ahead and ahead_ok:
                # Omega draw + sketch of the next block on a side stream: they overlap
                # this block's exchanges, panel and absorb
                o.sketch_async(self.rng, tt, b, self.Ys[tt % 2], prof=prof)
                return
            tok = prof.start("sketch_gemm")
            self._sketch_block(tt, self.Ys[tt % 2])
            prof.stop(tok)

        t = 0
        while True:
            sketch(t)
            if t > 0 and self.k + 2 * b <= self.max_rank:
                sketch(t + 1, ahead=True)  # look-ahead, issued before the exchanges
            tok = prof.start("schur_exchange")
            self._schur(self.Ys[t % 2])
            prof.stop(tok)
            if self.world > 1:
                e2, nc_prev, r_now, pmax = o.read(self.e2, self.meta[0:1], self.meta[1:2], self.meta[2:3])
            else:
                e2, nc_prev, r_now = o.read(self.e2, self.meta[0:1], self.meta[1:2])
            if pending:
                pending = False
                if nc_prev < b:  # zero pivot mid-block: redo the absorb truncated
                    self.cur, self.k = self._prev
                    self.scur = 1 - self.scur
                    self._absorb(nc_prev)
                    (self.r,) = o.read(self.meta[1:2])
                    status = STATUS_RANK_EXHAUSTED
                    break
            self.r = r_now
            if self.world > 1 and t > 0:
                self.pmax = pmax  # max count over ranks after the last absorb: pads the next all-gathers
            if t == 0:
                # adaptive_init (`skeleton.py:298-314`): full lupp of block 0
                if not math.isfinite(e2):
                    raise ValueError("matrix contains non-finite entries")
            else:
                e_schur = math.sqrt(e2) if e2 >= 0 else float("nan")
                trace.append(TraceRecord(k=self.k, e_schur=e_schur))
                if e_schur <= tau:
                    status = STATUS_OK
                    break
                if self.k + b > self.max_rank:
                    break
                if not math.isfinite(e2):
                    raise ValueError("matrix contains non-finite entries")
            R = m - self.k
            tok = prof.start("panel")
            o.panel(self.S[self.scur], R, b, self.sub, self.meta[0:1])
            prof.stop(tok)
            if t == 0:
                (nc,) = o.read(self.meta[0:1])
                if nc < b:
                    raise RankDeficientError(nc)
            tok = prof.start("absorb")
            self._absorb(b)
            prof.stop(tok)
            self.scur = 1 - self.scur  # the next Schur block goes to the other buffer
            pending = True
            t += 1
        return self._result(trace, status)

    def _result(self, trace, status):
        o = self.ops
        k = self.k
        mg = self.hi - self.lo
        W = o.f64(mg * k)
        o.scatter_interp_local(self.T[self.cur], k, self.perm[self.cur], self.loc, self.r, self.lo, self.hi, W)
        row_idx, w = o.output(self.perm[self.cur][:k].clone(), W[: mg * k].view(mg, k))
        return SkeletonResult(rank=k, row_idx=row_idx, w=w, trace=trace, status=status)
