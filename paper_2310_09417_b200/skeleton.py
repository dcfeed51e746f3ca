"""Randomized skeleton selection on the B200 -- drop-in for `randskel.skeleton`.

Entry points keep the reference signatures and results:
  rand_lupp(a, k, spec, rng)                          `skeleton.py:207-234`
  column_id(a, k, spec, rng)                          `skeleton.py:574-589`
  rand_lupp_adaptive(a, b, tau, spec, rng, max_rank)  `skeleton.py:391-460`
Sketch GEMMs, the panel LUPP, the Schur blocks, the interpolation update
and the W scatter run in librskel.so; Omega comes from the host RNG exactly
as in the reference.  Inputs may be numpy arrays (results come back as
numpy) or torch tensors (CUDA tensors stay on the device).
"""

import math
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _device, _engine, _lib, _omega, _ozaki, dense
from .errors import DimensionError, RankDeficientError
from .sketching import make_sketch

__all__ = [
    "STATUS_OK",
    "STATUS_NOT_CONVERGED",
    "STATUS_RANK_EXHAUSTED",
    "STATUS_ILL_CONDITIONED",
    "TraceRecord",
    "ErrorTrace",
    "SkeletonResult",
    "rand_lupp",
    "column_id",
    "rand_lupp_adaptive",
]

STATUS_OK = "ok"
STATUS_NOT_CONVERGED = "not_converged"
STATUS_RANK_EXHAUSTED = "rank_exhausted"
STATUS_ILL_CONDITIONED = "ill_conditioned"


@dataclass
class TraceRecord:
    """One adaptive iteration: rank so far and its error estimate."""

    k: int
    e_schur: float
    est_norm_ur: float | None = None
    est_max_ur: float | None = None


@dataclass
class ErrorTrace:
    """Per-iteration records with strictly increasing ranks (`skeleton.py:89-103`)."""

    records: list = field(default_factory=list)

    def append(self, record):
        if self.records and record.k <= self.records[-1].k:
            raise ValueError("trace ranks must be strictly increasing")
        self.records.append(record)

    def __len__(self):
        return len(self.records)

    def __iter__(self):
        return iter(self.records)


@dataclass
class SkeletonResult:
    """Outcome of a skeleton selection (`skeleton.py:106-129`).

    ``w`` interpolates rows (identity on ``row_idx``), ``x`` interpolates
    columns (identity on ``col_idx``)."""

    rank: int
    row_idx: object = None
    col_idx: object = None
    w: object = None
    x: object = None
    trace: ErrorTrace = field(default_factory=ErrorTrace)
    status: str = STATUS_OK

    @property
    def w_max(self):
        if self.w is None:
            return None
        if isinstance(self.w, torch.Tensor):
            return float(self.w.abs().max())
        return float(np.abs(self.w).max())


def _check_rank(k, m, n):
    if not 1 <= k <= min(m, n):
        raise DimensionError(f"k must be in [1, {min(m, n)}], got {k}")


def _factor_sketch(y, kind):
    """LUPP of a device sketch + interpolation matrix; raises like `lupp`."""
    m, ell = y.shape
    if m < ell:
        raise DimensionError(f"lupp requires rows >= cols, got {m} x {ell}")
    st, w, fail = _engine.factor_sample(y, want_w=True)
    if fail is not None:
        raise RankDeficientError(fail)
    return st, w


def _finite_or_raise(y, name="matrix"):
    e2 = torch.empty(1, dtype=torch.float64, device=y.t.device)
    from . import _lib
    _lib.call("rs_sumsq", y.ptr, y.ld, y.rows, y.cols, e2.data_ptr(),
              _device.workspace().data_ptr(), _device.stream_handle())
    if not math.isfinite(float(e2.item())):
        raise ValueError(f"{name} contains non-finite entries")


def _fixed_rank_sketch(a, sp, rng, transpose=False):
    """(device Matrix of a, Y) with Y = target @ Omega, target = a or a.T.
    Tensor-core engine: the target's digit planes (host input: cut as it
    lands) times Omega's; DMMA engine: the fp64 GEMM (host input: row chunks
    multiplied as they land)."""
    arr = _streamable(a)
    if _ozaki.sketch_engine() == "ozaki":
        om = _device.omega_dense(sp, rng)
        if arr is not None:
            tgt, planes = _streamed_planes(arr.T if transpose else arr)
            A = tgt.T if transpose else tgt
        else:
            A = _device.as_matrix(a)
            tgt = A.T if transpose else A
            planes = _ozaki.Planes.of_matrix(tgt)
        yt = torch.empty((tgt.rows, om.shape[1]), dtype=torch.float64, device=om.device)
        _ozaki.sketch(planes, _ozaki.Planes.of_omega(om), yt.data_ptr(), om.shape[1])
        if int(planes.nonfinite.item()):
            raise ValueError("matrix contains non-finite entries")
        return A, yt
    if arr is not None:  # H2D overlapped with the sketch, chunk by chunk
        return _streamed_sketch(arr, _device.omega_dense(sp, rng), transpose=transpose)
    A = _device.as_matrix(a)
    return A, _device.sketch_omega(A.T if transpose else A, sp, rng)


def rand_lupp(a, k, spec, rng):
    """Row skeletons by LUPP of ``a @ Omega`` (fixed rank k)."""
    m, n = _device.shape_of(a)
    _check_rank(k, m, n)
    sp = spec.with_dims(n, k)
    a, yt = _fixed_rank_sketch(a, sp, rng)
    y = _device.Matrix(yt, m, k, k, False, a.kind)
    _finite_or_raise(y)
    st, w = _factor_sketch(y, a.kind)
    idx = st.perm[:k].clone()
    return SkeletonResult(rank=k, row_idx=_device.to_host_index(idx, a.kind),
                          w=_device.to_output(w, a))


def column_id(a, k, spec, rng):
    """Column skeletons by LUPP of ``a.T @ Gamma``; ``x[:, col_idx] = I``."""
    m, n = _device.shape_of(a)
    _check_rank(k, m, n)
    sp = spec.with_dims(m, k)
    a, yt = _fixed_rank_sketch(a, sp, rng, transpose=True)
    y = _device.Matrix(yt, n, k, k, False, a.kind)
    _finite_or_raise(y)
    st, w = _factor_sketch(y, a.kind)
    idx = st.perm[:k].clone()
    x = _device.to_output(w, a)
    return SkeletonResult(rank=k, col_idx=_device.to_host_index(idx, a.kind), x=x.T)


def _checked_max_rank(m, n, b, tau, max_rank):
    if tau <= 0:
        raise ValueError(f"tau must be positive, got {tau}")
    if not 1 <= b <= min(m, n):
        raise DimensionError(f"block size must be in [1, {min(m, n)}], got {b}")
    if max_rank is None:
        max_rank = max(b, min(m, n) - b)
    return min(max_rank, min(m, n))


def _adaptive_device(A, b, tau, spec, rng, max_rank=None, planes=None):
    """`rand_lupp_adaptive` on a device Matrix, optionally with its digit
    planes already cut (cur.cur_decompose_adaptive reuses them)."""
    m, n = A.shape
    max_rank = _checked_max_rank(m, n, b, tau, max_rank)
    return _AdaptiveDriver(A, b, tau, rng, max_rank, spec=spec, planes=planes).run()


def rand_lupp_adaptive(a, b, tau, spec, rng, max_rank=None):
    """Adaptive blockwise LUPP row skeletons to absolute Frobenius tolerance tau.

    Block t sketches ``a @ Omega_t`` (Omega_t from ``rng.child(t)``), forms
    the Schur block against the current factorization, records its norm
    ``e_schur`` as the error estimate of the current rank, and stops at the
    first ``e_schur <= tau`` (status 'ok'), when ``rank + b > max_rank``
    ('not_converged'), or when a Schur block is exactly rank deficient
    ('rank_exhausted', truncated to the successful pivots).
    """
    m, n = _device.shape_of(a)
    if tau <= 0:
        raise ValueError(f"tau must be positive, got {tau}")
    if not 1 <= b <= min(m, n):
        raise DimensionError(f"block size must be in [1, {min(m, n)}], got {b}")
    if max_rank is None:
        max_rank = max(b, min(m, n) - b)
    max_rank = min(max_rank, min(m, n))
    if _ozaki.sketch_engine() == "ozaki":
        arr = _streamable(a)
        if arr is not None:  # H2D overlapped with the slicing of A into digit planes
            A, planes = _streamed_planes(arr)
            return _AdaptiveDriver(A, b, tau, rng, max_rank, spec=spec, planes=planes).run()
        return _AdaptiveDriver(_device.as_matrix(a), b, tau, rng, max_rank, spec=spec).run()
    pre = _presketch(a, b, rng, max_rank, spec)
    if pre is not None:
        A, yb, nb = pre
        return _AdaptiveDriver(A, b, tau, rng, max_rank, spec=spec, presketch=(yb, nb)).run()
    return _AdaptiveDriver(_device.as_matrix(a), b, tau, rng, max_rank, spec=spec).run()


_PRESKETCH_MIN_BYTES = 64 << 20
_PRESKETCH_MAX_BLOCKS = 32


def _streamable(a):
    """The host array behind ``a`` if its H2D can be overlapped with the
    sketch (fp64, C- or F-contiguous, >= 64 MB), else None."""
    import os

    if isinstance(a, (torch.Tensor, _device.Matrix)) or os.environ.get("RSKEL_PRESKETCH", "1") == "0":
        return None
    arr = np.asarray(a)
    if arr.dtype != np.float64 or arr.ndim != 2 or arr.nbytes < _PRESKETCH_MIN_BYTES:
        return None
    if not (arr.flags.c_contiguous or arr.flags.f_contiguous):
        return None
    return arr


def _streamed_sketch(arr, om, transpose=False):
    """Copy ``arr`` to the device in row chunks and accumulate
    ``target @ om`` (target = arr, or arr.T with ``transpose``) chunk by
    chunk as the rows land.  Returns (device Matrix of arr, Y tensor)."""
    dev = _device.device()
    m, n = arr.shape
    tm, tn = (n, m) if transpose else (m, n)   # target shape
    width = om.shape[1]
    Y = dense._mat(torch.empty((tm, width), dtype=torch.float64, device=dev))
    OM = dense._mat(om)
    a_colmajor = not arr.flags.c_contiguous
    under = arr.T if a_colmajor else arr       # C-ordered host rows
    t_colmajor = a_colmajor != transpose       # target's layout over `under`
    compute = torch.cuda.current_stream(dev)
    U = torch.empty(under.shape, dtype=torch.float64, device=dev)
    K = under.shape[0]
    # K-chunked accumulation (column-major target) in pieces aligned to the
    # GEMM's fixed chunks: the bits equal the one-shot product (rs_dgemm_ex)
    kc = _lib.load().rs_gemm_chunk(K) if t_colmajor else 1
    mode = 1 if kc < K else 2   # RS_GEMM_FOLD across chunks / RS_GEMM_CHAIN inside one

    def on_chunk(r0, r1, ev):
        compute.wait_event(ev)
        if t_colmajor:   # rows r0..r1 of `under` are columns (K) of the target
            A_part = _device.Matrix(U, tm, r1 - r0, tm, True, "numpy", off=r0 * tm)
            B_part = OM.sub(r0, 0, r1 - r0, width)
            _lib.call("rs_dgemm_ex", tm, width, r1 - r0, kc if kc < K else K, 0 if r0 == 0 else mode, 1.0,
                      A_part.ptr, A_part.ld, 1, None, B_part.ptr, B_part.ld, None, 0.0,
                      Y.ptr if r0 > 0 else None, Y.ld, None, Y.ptr, Y.ld, _device.workspace().data_ptr(),
                      _device.stream_handle())
        else:            # rows r0..r1 of `under` are rows of the target
            A_part = _device.Matrix(U, r1 - r0, tn, tn, False, "numpy", off=r0 * tn)
            dense._gemm(Y.sub(r0, 0, r1 - r0, width), A_part, OM)

    _device.h2d_rows(under, on_chunk, out=U, align=kc)
    A = _device.Matrix(U, m, n, m if a_colmajor else n, a_colmajor, "numpy")
    return A, Y.t


def _streamed_planes(arr):
    """Copy the host array to the device in chunks and cut every chunk into
    the tensor-core sketch's digit planes as it lands (the copy engine and
    the slicing kernels overlap).  Chunks are aligned to the planes' K-chunks
    (column-major candidates) or row tiles, so the planes -- and every sketch
    bit -- equal those of a device-resident A."""
    dev = _device.device()
    m, n = arr.shape
    a_colmajor = not arr.flags.c_contiguous
    under = arr.T if a_colmajor else arr       # C-ordered host rows
    U = torch.empty(under.shape, dtype=torch.float64, device=dev)
    planes = _ozaki.Planes(m, n, _ozaki.A_PLANES[torch.float64], 128, dev)
    compute = torch.cuda.current_stream(dev)

    def on_chunk(r0, r1, ev):
        compute.wait_event(ev)
        if a_colmajor:   # rows r0..r1 of `under` are K-columns r0..r1 of the candidates
            planes.fill(U.data_ptr(), False, m, True, r0, r1)
        else:            # rows r0..r1 of `under` are candidate rows
            planes.fill_rows(U.data_ptr() + 8 * r0 * n, False, n, r0, r1)

    _device.h2d_rows(under, on_chunk, out=U, align=planes.kc if a_colmajor else 128)
    A = _device.Matrix(U, m, n, m if a_colmajor else n, a_colmajor, "numpy")
    return A, planes


def _presketch(a, b, rng, max_rank, spec):
    """Host input: overlap the H2D of A with the sketches of the first blocks.

    One wide product A-side x [Omega_0 | ... | Omega_{NB-1}] is accumulated
    over row chunks of the host array as they land on the device, so the
    copy engine and the DMMA pipe work at the same time; the loop then starts
    with NB sketch blocks already computed.  Returns None when not
    applicable (device input, small input, non-Gaussian or host draws)."""
    if spec.kind != "gaussian" or _device.host_rng() or b > _engine.MAX_BLOCK:
        return None
    arr = _streamable(a)
    if arr is None:
        return None
    m, n = arr.shape
    nb = min(_PRESKETCH_MAX_BLOCKS, max_rank // b + 1)
    if nb < 2:
        return None
    dev = _device.device()
    om = torch.empty((n, b * nb), dtype=torch.float64, device=dev)
    for t in range(nb):
        om[:, b * t: b * (t + 1)].copy_(_device.gaussian(rng.child(t), n, b))
    A, yb = _streamed_sketch(arr, om)
    return A, yb, nb


# experiment switch: RSKEL_LOOKAHEAD=0 sketches block t + 1 on the compute stream
# instead of beside block t's panel and absorb
import os as _os  # noqa: E402

_LOOKAHEAD = _os.environ.get("RSKEL_LOOKAHEAD", "1") != "0"


class _BlockOperators:
    """SRTT / sparse-sign block operators (the reference's per-block draw,
    `skeleton.py:286-295`) drawn ahead on the host thread pool: numpy releases
    the GIL in the uniform fill and the argsort, so the draws of the next
    blocks (~30 ms each for a 20000 x 64 sparse sign) overlap each other and
    the device work of the current block.  Same operators, same order."""

    def __init__(self, spec, n, b, rng, nblocks, depth=None):
        import os

        from . import _omega
        from .lu_state import _block_spec

        if depth is None:  # blocks drawn ahead (RSKEL_OPS_AHEAD=1: the current block only)
            depth = int(os.environ.get("RSKEL_OPS_AHEAD", "8"))

        self.sp, self.rng, self.nblocks, self.depth = _block_spec(spec, n, b), rng, nblocks, depth
        self.pool = _omega._pool()
        self.fut = {}

    def get(self, t):
        for u in range(t, min(self.nblocks, t + self.depth)):
            if u not in self.fut:
                self.fut[u] = self.pool.submit(make_sketch, self.sp, self.rng.child(u))
        f = self.fut.pop(t, None)
        return f.result() if f is not None else make_sketch(self.sp, self.rng.child(t))

    def close(self):
        for f in self.fut.values():
            f.cancel()
        self.fut.clear()


class PhaseTimer:
    """Optional CUDA-event instrumentation of the adaptive loop phases
    (sketch / schur / panel / absorb / interp), used by bench.py for the
    roofline of the dominant kernel.  Events are recorded on the launching
    stream; ``totals()`` syncs and returns milliseconds per phase."""

    def __init__(self):
        self.events = {}
        self.counts = {}

    def start(self, name):
        ev = torch.cuda.Event(enable_timing=True)
        ev.record()
        return (name, ev)

    def stop(self, token):
        name, ev0 = token
        ev1 = torch.cuda.Event(enable_timing=True)
        ev1.record()
        self.events.setdefault(name, []).append((ev0, ev1))

    def totals(self):
        torch.cuda.synchronize()
        return {k: sum(a.elapsed_time(b) for a, b in v) for k, v in self.events.items()}

    def launches(self):
        return {k: len(v) for k, v in self.events.items()}


_PHASE_TIMER = None  # set to a PhaseTimer to instrument rand_lupp_adaptive


class _NullTimer:
    def start(self, name):
        return None

    def stop(self, token):
        pass


class _AdaptiveDriver:
    """Host side of the adaptive loop.

    Streams: Omega_t is copied H2D on a side stream into a double-buffered
    device slot while the compute stream works on earlier blocks; the sketch
    of block t+1 is enqueued before the host waits for block t's estimate, and
    the absorb of a block is enqueued speculatively (assuming a full-width
    elimination) before its eliminated-column count is read back.  The host
    therefore waits once per block (e2 of block t plus ncols of block t-1 in
    one pinned readback) while the GPU keeps the next sketch GEMM running.
    """

    def __init__(self, a, b, tau, rng, max_rank, host=False, spec=None, presketch=None, planes=None):
        self.prof = _PHASE_TIMER or _NullTimer()
        self.a, self.b, self.tau, self.rng, self.max_rank = a, b, tau, rng, max_rank
        m, n = a.shape
        self.m, self.n = m, n
        dev = _device.device()
        # Omega_t: device draw (rs_gaussian) on the side stream by default,
        # host thread-pool draw + H2D copy under RSKEL_HOST_RNG=1.
        self.spec = spec
        self.kind = spec.kind if spec is not None else "gaussian"
        # blocks t < nb_pre were sketched during the H2D (`_presketch`)
        self.yb, self.nb_pre = presketch if presketch is not None else (None, 0)
        self.dev_rng = not (host or _device.host_rng())
        self.src = None if (self.dev_rng or self.kind != "gaussian") else _omega.BlockOmegaSource(n, b, rng)
        self.rng_status = torch.zeros(max(max_rank, b) // b + 4, dtype=torch.int32, device=dev)
        self.ops_ahead = (None if self.kind == "gaussian" else
                          _BlockOperators(spec, n, b, rng, self.rng_status.numel()))
        self.om = [torch.empty((n, b), dtype=torch.float64, device=dev) for _ in range(2)]
        self.y = [torch.empty((m, b), dtype=torch.float64, device=dev) for _ in range(2)]
        self.om_ready = [torch.cuda.Event() for _ in range(2)]
        self.om_free = [None, None]
        self.copy_stream = torch.cuda.Stream(device=dev)
        self.compute = torch.cuda.current_stream(dev)
        if self.dev_rng:
            _device._rng_workspace(n * b)       # allocated on the compute stream
        self.copy_stream.wait_stream(self.compute)  # prior users of the RNG workspace
        self.e2 = torch.empty(1, dtype=torch.float64, device=dev)
        self.nc = torch.empty(max(1, (b + 63) // 64), dtype=torch.int32, device=dev)
        self.h_e2 = torch.empty(1, dtype=torch.float64, pin_memory=True)
        self.h_nc = torch.empty(1, dtype=torch.int32, pin_memory=True)
        # the first block is always absorbed whole (adaptive_init), so the
        # rank can reach b even when max_rank < b (`skeleton.py:435-441`)
        self.st = _engine.TFormState(m, max(max_rank, b), min(b, _engine.MAX_BLOCK))
        # tensor-core sketch: A's digit planes once, Omega_t's per block
        self.ozaki = _ozaki.sketch_engine() == "ozaki" and self.yb is None and self.kind != "sparsesign"
        if self.kind == "sparsesign":  # the look-ahead SpMM's stream
            self.sketch_stream = torch.cuda.Stream(device=dev)
        if self.ozaki:
            tok = self.prof.start("a_slice")
            self.ap = planes if planes is not None else _ozaki.Planes.of_matrix(a)
            self.prof.stop(tok)
            self.bp = _ozaki.Planes(b, n, _ozaki.OMEGA_PLANES, 64, dev)
            self.sketch_stream = torch.cuda.Stream(device=dev)
            self.ws_ahead = _device.workspace(slot=1)
        self.y_ready = [None, None]
        # a large numpy W: its pages are faulted in while the loop runs (host idle)
        self.w_host = None
        if a.kind == "numpy" and 8 * m * max(max_rank, b) >= (256 << 20):
            self.w_host = _device.HostPrefault(8 * m * max(max_rank, b))
        self.stream = _device.stream_handle()
        self.ws = _device.workspace()
        self._issued = set()

    # -- Omega pipeline --------------------------------------------------------
    def _issue_copy(self, t):
        if t in self._issued or self.kind == "sparsesign":
            return
        self._issued.add(t)
        slot = t % 2
        if t >= self.rng_status.numel():
            return
        h = None if (self.dev_rng or self.kind != "gaussian") else self.src.host(t)
        with torch.cuda.stream(self.copy_stream):
            if self.om_free[slot] is not None:
                self.copy_stream.wait_event(self.om_free[slot])
            if self.kind != "gaussian":
                # SRTT: the reference's per-block operator (`skeleton.py:286-295`), dense on the device
                self.om[slot].copy_(self.ops_ahead.get(t).device_dense())
            elif h is None:
                _device.gaussian(self.rng.child(t), self.n, self.b, out=self.om[slot],
                                 status=self.rng_status[t:t + 1])
            else:
                self.om[slot].copy_(h, non_blocking=True)
            self.om_ready[slot].record(self.copy_stream)

    def _y(self, t):
        """(pointer, leading dimension) of block t's sketch."""
        if t < self.nb_pre:
            return self.yb.data_ptr() + 8 * self.b * t, self.b * self.nb_pre
        return self.y[t % 2].data_ptr(), self.b

    def _sketch(self, t, ahead=False):
        """Sketch of block t into Y slot t % 2.  ``ahead``: the look-ahead block
        on the tensor cores, on its own stream and workspace, so it runs beside
        the current block's panel and absorb (`_wait_y` joins before use)."""
        from . import _lib
        if t < self.nb_pre:
            return
        slot = t % 2
        if self.kind == "sparsesign":
            # the reference's per-block operator (`skeleton.py:286-295`) applied as an
            # SpMM (Y_t bitwise the reference's); the look-ahead block on its own stream,
            # where its small CTAs can share the SMs with the cooperative panel
            op = self.ops_ahead.get(t)
            if ahead and _LOOKAHEAD:
                ss = self.sketch_stream
                ss.wait_stream(self.compute)  # the slot's previous readers
                with torch.cuda.stream(ss):
                    _device.sparse_sign_apply(self.a, op.idx, op.signs, op.ell, op.scale, out=self.y[slot])
                    ev = torch.cuda.Event()
                    ev.record(ss)
                self.y_ready[slot] = ev
                return
            tok = self.prof.start("sketch_gemm")
            _device.sparse_sign_apply(self.a, op.idx, op.signs, op.ell, op.scale, out=self.y[slot])
            self.prof.stop(tok)
            self.y_ready[slot] = None
            return
        self._issue_copy(t)
        if ahead and self.ozaki and _LOOKAHEAD:
            ss = self.sketch_stream
            ss.wait_stream(self.compute)        # the slot's previous readers are enqueued on compute
            ss.wait_event(self.om_ready[slot])
            with torch.cuda.stream(ss):
                tok = self.prof.start("omega_slice")
                _ozaki.Planes.of_omega(self.om[slot], out=self.bp, ws=self.ws_ahead)
                self.prof.stop(tok)
                tok = self.prof.start("sketch_gemm")
                _ozaki.sketch(self.ap, self.bp, self.y[slot].data_ptr(), self.b, ws=self.ws_ahead)
                self.prof.stop(tok)
                ev = torch.cuda.Event()
                ev.record(ss)
            self.y_ready[slot] = ev
            self.om_free[slot] = ev
            self._issue_copy(t + 2)
            return
        self.compute.wait_event(self.om_ready[slot])
        if self.ozaki:
            tok = self.prof.start("omega_slice")
            _ozaki.Planes.of_omega(self.om[slot], out=self.bp)
            self.prof.stop(tok)
            tok = self.prof.start("sketch_gemm")
            _ozaki.sketch(self.ap, self.bp, self.y[slot].data_ptr(), self.b)
        else:
            tok = self.prof.start("sketch_gemm")
            _lib.call("rs_sketch_gemm", self.m, self.n, self.b, self.a.ptr, self.a.ld, int(self.a.colmajor),
                      self.om[slot].data_ptr(), self.b, self.y[slot].data_ptr(), self.b,
                      self.ws.data_ptr(), self.stream)
        self.prof.stop(tok)
        ev = torch.cuda.Event()
        ev.record(self.compute)
        self.om_free[slot] = ev
        self.y_ready[slot] = None
        self._issue_copy(t + 2)

    def _wait_y(self, t):
        if t >= self.nb_pre and self.y_ready[t % 2] is not None:
            self.compute.wait_event(self.y_ready[t % 2])

    # -- blocks ------------------------------------------------------------------
    def _absorb_block(self, y, first):
        """Eliminate the current block synchronously (first block, and b > 64);
        returns eliminated columns (< b iff a zero pivot column, `_lupp_partial`).
        ``y`` = (pointer, leading dimension) of the block's sketch."""
        st, b = self.st, self.b
        yp, ld = y
        done = 0
        for j0 in range(0, b, _engine.MAX_BLOCK):
            w = min(_engine.MAX_BLOCK, b - j0)
            if j0 > 0 or first or b > _engine.MAX_BLOCK:
                st.schur(yp + 8 * j0, ld, w, None)
            st.panel(w, self.nc)
            nc = int(self.nc[0].item())
            st.absorb(w, nc)
            done += nc
            if nc < w:
                break
        return done

    def _readback(self, with_nc):
        self.h_e2.copy_(self.e2, non_blocking=True)
        if with_nc:
            self.h_nc.copy_(self.nc[:1], non_blocking=True)
        ev = torch.cuda.Event()
        ev.record(self.compute)
        return ev

    def run(self):
        st, b, tau = self.st, self.b, self.tau
        wide = b > _engine.MAX_BLOCK
        try:
            # adaptive_init (`skeleton.py:298-314`): lupp of the first block.
            self._sketch(0)
            y0 = self._y(0)
            st.schur(y0[0], y0[1], min(b, _engine.MAX_BLOCK), self.e2)
            if self.ozaki and int(self.ap.nonfinite.item()):
                raise ValueError("matrix contains non-finite entries")
            if wide or not math.isfinite(float(self.e2.item())):
                if self.nb_pre:
                    _finite_or_raise(_device.Matrix(self.yb, self.m, b, b * self.nb_pre, False, self.a.kind))
                else:
                    _finite_or_raise(_device.Matrix(self.y[0], self.m, b, b, False, self.a.kind))
            done = self._absorb_block(y0, first=True)
            if done < b:
                raise RankDeficientError(done)
            trace = ErrorTrace()
            status = STATUS_NOT_CONVERGED
            t = 1
            self._sketch(1, ahead=not wide)
            pending = False  # speculative full-width absorb awaiting its ncols
            # b == 64: absorb(t) and the Schur block of t+1 run as one fused
            # pass over T (rs_absorb_schur); S/e2 of block t are then ready.
            fused = b == _engine.MAX_BLOCK
            have_schur = False
            while True:
                y = self._y(t)
                self._wait_y(t)
                if not wide and not have_schur:
                    tok = self.prof.start("schur")
                    st.schur(y[0], y[1], b, self.e2)
                    self.prof.stop(tok)
                if wide:
                    e2 = 0.0
                    for j0 in range(0, b, _engine.MAX_BLOCK):
                        w = min(_engine.MAX_BLOCK, b - j0)
                        st.schur(y[0] + 8 * j0, y[1], w, self.e2)
                        e2 += float(self.e2.item())
                    ev = None
                else:
                    ev = self._readback(pending)
                # speculative: next block's sketch runs while the host waits (tensor-core
                # engine: on its own stream, beside this block's panel and absorb)
                self._sketch(t + 1, ahead=not wide)
                if ev is not None:
                    ev.synchronize()
                    e2 = float(self.h_e2[0])
                if pending:
                    nc_prev = int(self.h_nc[0])
                    pending = False
                    if nc_prev < b:  # zero pivot mid-block: redo the absorb truncated
                        st.rollback()
                        st.absorb(b, nc_prev)
                        status = STATUS_RANK_EXHAUSTED
                        break
                e_schur = math.sqrt(e2) if e2 >= 0 else float("nan")
                trace.append(TraceRecord(k=st.k, e_schur=e_schur))
                if e_schur <= tau:
                    status = STATUS_OK
                    break
                if st.k + b > self.max_rank:
                    break
                if not math.isfinite(e2):
                    raise ValueError("matrix contains non-finite entries")
                if self.w_host is not None:
                    self.w_host.advance(8 * self.m * (st.k + 2 * b))
                if not wide:
                    tok = self.prof.start("panel")
                    st.panel(b, self.nc)
                    self.prof.stop(tok)
                    tok = self.prof.start("absorb")
                    if fused:
                        yn = self._y(t + 1)
                        st.absorb(b, b)
                        self._wait_y(t + 1)
                        st.schur_next(yn[0], yn[1], self.e2)  # into the other S buffer (rollback keeps S)
                        have_schur = True
                    else:
                        st.absorb(b, b)
                    self.prof.stop(tok)
                    pending = True
                    nc = b
                else:
                    nc = self._absorb_block(y, first=False)
                t += 1
                if nc < b:
                    status = STATUS_RANK_EXHAUSTED
                    break
        except BaseException:
            if self.w_host is not None:
                self.w_host.close()
            raise
        finally:
            if self.src is not None:
                self.src.close()
            if self.ops_ahead is not None:
                self.ops_ahead.close()
            # speculative draws / sketches may still be in flight on the side streams
            self.compute.wait_stream(self.copy_stream)
            if self.ozaki or self.kind == "sparsesign":
                self.compute.wait_stream(self.sketch_stream)
        if self.dev_rng and bool(self.rng_status.any()):
            # a block the parallel ziggurat resolver could not place (never
            # observed): redo the whole loop with the host draw, same bits
            self.dev_rng = False
            if self.w_host is not None:
                self.w_host.close()
            self.__init__(self.a, self.b, self.tau, self.rng, self.max_rank, host=True, spec=self.spec)
            # (the presketched blocks are dropped: every block is redrawn on the host)
            return self.run()
        k = st.k
        tok = self.prof.start("interp")
        w = st.interpolation()
        self.prof.stop(tok)
        kind = self.a.kind
        return SkeletonResult(rank=k, row_idx=_device.to_host_index(st.perm[:k].clone(), kind),
                              w=_device.to_output(w, kind, host_out=self.w_host), trace=trace, status=status)
