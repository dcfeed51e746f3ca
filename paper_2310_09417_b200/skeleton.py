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

from . import _device, _engine, _omega
from .errors import DimensionError, RankDeficientError
from .sketching import make_gaussian, make_sketch

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


def rand_lupp(a, k, spec, rng):
    """Row skeletons by LUPP of ``a @ Omega`` (fixed rank k)."""
    a = _device.as_matrix(a)
    m, n = a.shape
    _check_rank(k, m, n)
    op = make_sketch(spec.with_dims(n, k), rng)
    y = _device.Matrix(_device.sketch(a, op.omega), m, k, k, False, a.kind)
    _finite_or_raise(y)
    st, w = _factor_sketch(y, a.kind)
    idx = st.perm[:k].clone()
    return SkeletonResult(rank=k, row_idx=_device.to_host_index(idx, a.kind),
                          w=_device.to_output(w, a))


def column_id(a, k, spec, rng):
    """Column skeletons by LUPP of ``a.T @ Gamma``; ``x[:, col_idx] = I``."""
    a = _device.as_matrix(a)
    m, n = a.shape
    _check_rank(k, m, n)
    op = make_sketch(spec.with_dims(m, k), rng)
    y = _device.Matrix(_device.sketch(a.T, op.omega), n, k, k, False, a.kind)
    _finite_or_raise(y)
    st, w = _factor_sketch(y, a.kind)
    idx = st.perm[:k].clone()
    x = _device.to_output(w, a)
    return SkeletonResult(rank=k, col_idx=_device.to_host_index(idx, a.kind), x=x.T)


def rand_lupp_adaptive(a, b, tau, spec, rng, max_rank=None):
    """Adaptive blockwise LUPP row skeletons to absolute Frobenius tolerance tau.

    Block t sketches ``a @ Omega_t`` (Omega_t from ``rng.child(t)``), forms
    the Schur block against the current factorization, records its norm
    ``e_schur`` as the error estimate of the current rank, and stops at the
    first ``e_schur <= tau`` (status 'ok'), when ``rank + b > max_rank``
    ('not_converged'), or when a Schur block is exactly rank deficient
    ('rank_exhausted', truncated to the successful pivots).
    """
    a = _device.as_matrix(a)
    m, n = a.shape
    if tau <= 0:
        raise ValueError(f"tau must be positive, got {tau}")
    if not 1 <= b <= min(m, n):
        raise DimensionError(f"block size must be in [1, {min(m, n)}], got {b}")
    if max_rank is None:
        max_rank = max(b, min(m, n) - b)
    max_rank = min(max_rank, min(m, n))
    if spec.kind != "gaussian":
        make_sketch(spec.with_dims(n, b), rng)  # raises NotImplementedError
    return _AdaptiveDriver(a, b, tau, rng, max_rank).run()


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
    """Host side of the adaptive loop: one Omega block H2D, one e2 D2H and one
    eliminated-column count D2H per block; everything else on the device."""

    def __init__(self, a, b, tau, rng, max_rank):
        self.prof = _PHASE_TIMER or _NullTimer()
        self.a, self.b, self.tau, self.rng, self.max_rank = a, b, tau, rng, max_rank
        m, n = a.shape
        self.m, self.n = m, n
        dev = _device.device()
        self.src = _omega.BlockOmegaSource(n, b, rng)
        self.om = torch.empty((n, b), dtype=torch.float64, device=dev)
        self.y = torch.empty((m, b), dtype=torch.float64, device=dev)
        self.e2 = torch.empty(1, dtype=torch.float64, device=dev)
        self.nc = torch.empty(max(1, (b + 63) // 64), dtype=torch.int32, device=dev)
        self.st = _engine.TFormState(m, max_rank, min(b, _engine.MAX_BLOCK))
        self.stream = _device.stream_handle()

    def _sketch(self, t):
        from . import _lib
        h = self.src.host(t)
        tok = self.prof.start("omega_h2d")
        self.om.copy_(h, non_blocking=True)
        self.prof.stop(tok)
        tok = self.prof.start("sketch_gemm")
        _lib.call("rs_sketch_gemm", self.m, self.n, self.b, self.a.ptr, self.a.ld, int(self.a.colmajor),
                  self.om.data_ptr(), self.b, self.y.data_ptr(), self.b, self.stream)
        self.prof.stop(tok)

    def _schur_norm2(self):
        """||Y[perm[k:]] - T Y[perm[:k]]||^2 over all b columns (current state)."""
        st, b = self.st, self.b
        if b <= _engine.MAX_BLOCK:
            tok = self.prof.start("schur")
            st.schur(self.y.data_ptr(), b, b, self.e2)
            self.prof.stop(tok)
            return float(self.e2.item())
        total = 0.0
        for j0 in range(0, b, _engine.MAX_BLOCK):
            w = min(_engine.MAX_BLOCK, b - j0)
            st.schur(self.y.data_ptr() + 8 * j0, b, w, self.e2)
            total += float(self.e2.item())
        return total

    def _absorb_block(self, first):
        """Eliminate the current block; returns eliminated columns (< b iff an
        exactly-zero pivot column was met, `_lupp_partial`)."""
        st, b = self.st, self.b
        done = 0
        for j0 in range(0, b, _engine.MAX_BLOCK):
            w = min(_engine.MAX_BLOCK, b - j0)
            if j0 > 0 or first or b > _engine.MAX_BLOCK:
                st.schur(self.y.data_ptr() + 8 * j0, b, w, None)
            st.panel(w, self.nc)
            nc = int(self.nc[0].item())
            st.absorb(w, nc)
            done += nc
            if nc < w:
                break
        return done

    def run(self):
        st, b, tau = self.st, self.b, self.tau
        try:
            # adaptive_init (`skeleton.py:298-314`): lupp of the first block.
            self._sketch(0)
            st.schur(self.y.data_ptr(), b, min(b, _engine.MAX_BLOCK), self.e2)
            if b > _engine.MAX_BLOCK or not math.isfinite(float(self.e2.item())):
                _finite_or_raise(_device.Matrix(self.y, self.m, b, b, False, self.a.kind))
            done = self._absorb_block(first=True)
            if done < b:
                raise RankDeficientError(done)
            trace = ErrorTrace()
            status = STATUS_NOT_CONVERGED
            t = 1
            while True:
                self._sketch(t)
                e2 = self._schur_norm2()
                e_schur = math.sqrt(e2) if e2 >= 0 else float("nan")
                trace.append(TraceRecord(k=st.k, e_schur=e_schur))
                if e_schur <= tau:
                    status = STATUS_OK
                    break
                if st.k + b > self.max_rank:
                    break
                if not math.isfinite(e2):
                    raise ValueError("matrix contains non-finite entries")
                if b <= _engine.MAX_BLOCK:
                    tok = self.prof.start("panel")
                    st.panel(b, self.nc)
                    self.prof.stop(tok)
                    nc = int(self.nc[0].item())
                    tok = self.prof.start("absorb")
                    st.absorb(b, nc)
                    self.prof.stop(tok)
                else:
                    nc = self._absorb_block(first=False)
                t += 1
                if nc < b:
                    status = STATUS_RANK_EXHAUSTED
                    break
        finally:
            self.src.close()
        k = st.k
        tok = self.prof.start("interp")
        w = st.interpolation()
        self.prof.stop(tok)
        kind = self.a.kind
        return SkeletonResult(rank=k, row_idx=_device.to_host_index(st.perm[:k].clone(), kind),
                              w=_device.to_output(w, kind), trace=trace, status=status)
