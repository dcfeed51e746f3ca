"""Device plumbing: matrix descriptors, host<->device transfer, streams and
workspaces.  PyTorch is used only to own device/pinned memory and streams;
all arithmetic on the skeleton path goes through librskel.so.

Ownership mirrors the reference (`dense.py:52-62`): inputs are converted to
float64 and never mutated; outputs are fresh arrays.  Results come back in
the caller's container: numpy in -> numpy out, torch CPU -> torch CPU, torch
CUDA -> torch CUDA (device-resident, no D2H).
"""

import numpy as np
import torch

from . import _lib
from .errors import DeviceError, DimensionError

_workspaces = {}


def device():
    if not torch.cuda.is_available():
        raise DeviceError("no CUDA device visible: the skeleton path runs on B200 only (no CPU fallback)")
    return torch.device("cuda", torch.cuda.current_device())


def stream_handle():
    return torch.cuda.current_stream().cuda_stream


def workspace(slot=0):
    """The library scratch of this device; ``slot`` > 0 gives separate
    workspaces for work enqueued concurrently on other streams."""
    dev = device()
    ws = _workspaces.get((dev.index, slot))
    if ws is None:
        ws = torch.zeros(_lib.load().rs_workspace_bytes(), dtype=torch.uint8, device=dev)  # GEMM counters start at 0
        _workspaces[(dev.index, slot)] = ws
    return ws


class Matrix:
    """fp64 device matrix view.  Element (i, j) lives at ``base[i*ld + j]``
    (row-major) or ``base[j*ld + i]`` (column-major).  ``kind`` records the
    caller's container so results can be returned the same way."""

    __slots__ = ("t", "rows", "cols", "ld", "colmajor", "kind", "off", "src32")

    def __init__(self, t, rows, cols, ld, colmajor, kind, off=0):
        self.t, self.rows, self.cols, self.ld, self.colmajor, self.kind = t, rows, cols, ld, colmajor, kind
        self.off = off  # element offset of (0, 0) from t.data_ptr()
        # fp32 input: the caller's values as fp32 on the device (same layout and ld),
        # read directly by the tensor-core sketch; t holds the exact fp64 upcast
        self.src32 = None

    @property
    def ptr(self):
        return self.t.data_ptr() + 8 * self.off

    @property
    def shape(self):
        return (self.rows, self.cols)

    @property
    def T(self):
        m = Matrix(self.t, self.cols, self.rows, self.ld, not self.colmajor, self.kind, self.off)
        m.src32 = self.src32.T if self.src32 is not None else None
        return m

    def sub(self, r0, c0, rows, cols):
        """View of the block [r0:r0+rows, c0:c0+cols] (no copy)."""
        off = self.off + (c0 * self.ld + r0 if self.colmajor else r0 * self.ld + c0)
        return Matrix(self.t, rows, cols, self.ld, self.colmajor, self.kind, off)

    def tensor(self):
        """The block as a strided torch view."""
        st = (1, self.ld) if self.colmajor else (self.ld, 1)
        return torch.as_strided(self.t, (self.rows, self.cols), st, self.t.storage_offset() + self.off)

    def row_major(self):
        """A row-major view of the same matrix (device transpose copy if needed)."""
        if not self.colmajor:
            return self
        out = torch.empty((self.rows, self.cols), dtype=torch.float64, device=self.t.device)
        if self.rows and self.cols:
            _lib.call("rs_transpose", self.ptr, self.ld, self.cols, self.rows, out.data_ptr(),
                      self.cols, stream_handle())
        return Matrix(out, self.rows, self.cols, self.cols, False, self.kind)

    def copy(self):
        """Fresh row-major copy (device kernels only)."""
        src = self.row_major()
        if src is not self:
            return src
        out = torch.empty((self.rows, self.cols), dtype=torch.float64, device=self.t.device)
        if self.rows and self.cols:
            _lib.call("rs_gather_rows", self.ptr, self.ld, None, self.rows, self.cols, out.data_ptr(),
                      max(self.cols, 1), stream_handle())
        return Matrix(out, self.rows, self.cols, max(self.cols, 1), False, self.kind)


def empty(rows, cols, kind="torch_cuda"):
    t = torch.empty((rows, cols), dtype=torch.float64, device=device())
    return Matrix(t, rows, cols, max(cols, 1), False, kind)


def _from_tensor_2d(t, kind):
    rows, cols = t.shape
    s0, s1 = t.stride()
    if rows == 0 or cols == 0:
        t = t.contiguous()
        return Matrix(t, rows, cols, max(cols, 1), False, kind)
    if s1 == 1 and (rows == 1 or s0 >= cols):
        return Matrix(t, rows, cols, s0 if rows > 1 else cols, False, kind)
    if s0 == 1 and (cols == 1 or s1 >= rows):
        return Matrix(t, rows, cols, s1 if cols > 1 else rows, True, kind)
    t = t.contiguous()
    return Matrix(t, rows, cols, cols, False, kind)


def shape_of(a, name="matrix"):
    """(m, n) of a matrix-like without touching the device; DimensionError if
    it is not 2-D (mirrors `_require_2d`, skeleton.py:200-204)."""
    if isinstance(a, Matrix):
        return a.shape
    shp = tuple(a.shape) if hasattr(a, "shape") else np.shape(a)
    if len(shp) != 2:
        raise DimensionError(f"{name} must be 2-dimensional, got shape {shp}")
    return shp


def as_matrix(a, name="matrix"):
    """Convert ``a`` (numpy / array_like / torch / Matrix) to an fp64 device Matrix."""
    if isinstance(a, Matrix):
        return a
    dev = device()
    if isinstance(a, torch.Tensor):
        if a.dim() != 2:
            raise DimensionError(f"{name} must be 2-dimensional, got shape {tuple(a.shape)}")
        kind = "torch_cuda" if a.is_cuda else "torch_cpu"
        if not a.is_cuda:
            if a.dtype not in (torch.float32, torch.float64):
                a = a.to(torch.float64)
            if a.t().is_contiguous() and not a.is_contiguous():
                a = h2d(a.t().numpy()).t()
            else:
                a = h2d(a.contiguous().numpy())
        a32 = a if a.dtype == torch.float32 else None
        if a.dtype != torch.float64:
            a = a.to(torch.float64)
        m = _from_tensor_2d(a, kind)
        if a32 is not None:
            m.src32 = _from_tensor_2d(a32, kind)
            if (m.src32.colmajor, m.src32.ld) != (m.colmajor, m.ld):  # layouts must agree
                m.src32 = None
        return m
    arr = np.asarray(a)
    if arr.dtype not in (np.float32, np.float64):
        arr = arr.astype(np.float64)
    if arr.ndim != 2:
        raise DimensionError(f"{name} must be 2-dimensional, got shape {arr.shape}")
    if not (arr.flags.c_contiguous or arr.flags.f_contiguous):
        arr = np.ascontiguousarray(arr)
    colmajor = not arr.flags.c_contiguous
    t = h2d(arr.T if colmajor else arr)
    t32 = None
    if t.dtype != torch.float64:  # fp32 input: upcast on the device (half the H2D bytes)
        t32 = t
        t = t.to(torch.float64)
    rows, cols = arr.shape
    ld = max(rows if colmajor else cols, 1)
    m = Matrix(t, rows, cols, ld, colmajor, "numpy")
    if t32 is not None:
        m.src32 = Matrix(t32, rows, cols, ld, colmajor, "numpy")
    return m


# ------------------------------------------------------------- host -> device --
_STAGE_BYTES = 32 << 20
_STAGE_DEPTH = 4
_stage = {}


def _stage_ring(dev):
    ring = _stage.get(dev.index)
    if ring is None:
        ring = {
            "bufs": [torch.empty(_STAGE_BYTES, dtype=torch.uint8, pin_memory=True) for _ in range(_STAGE_DEPTH)],
            "events": [None] * _STAGE_DEPTH,
            "stream": torch.cuda.Stream(device=dev),
        }
        _stage[dev.index] = ring
    return ring


def _copy_pool():
    from . import _omega
    return _omega._pool()


def h2d(arr):
    """Device copy of a C-contiguous host array.  Page-locked memory goes
    straight to DMA; pageable memory (a user's numpy array) is staged through
    a ring of pinned 32 MB chunks that host threads fill while earlier chunks
    are in flight, instead of the driver's synchronous pageable path."""
    dev = device()
    host = torch.from_numpy(arr)
    nbytes = arr.nbytes
    if nbytes < (8 << 20) or host.is_pinned():
        return host.to(dev, non_blocking=host.is_pinned())
    out = torch.empty(arr.shape, dtype=host.dtype, device=dev)
    src = arr.reshape(-1).view(np.uint8)
    dst = out.view(-1).view(torch.uint8)
    ring = _stage_ring(dev)
    pool = _copy_pool()
    nthr = max(1, min(16, pool._max_workers))
    cs = ring["stream"]
    cs.wait_stream(torch.cuda.current_stream(dev))  # `out` was allocated on the compute stream
    for i, c0 in enumerate(range(0, nbytes, _STAGE_BYTES)):
        c1 = min(nbytes, c0 + _STAGE_BYTES)
        slot = i % _STAGE_DEPTH
        ev = ring["events"][slot]
        if ev is not None:
            ev.synchronize()
        buf = ring["bufs"][slot].numpy()
        step = -(-(c1 - c0) // nthr)
        parts = [(p0, min(c1 - c0, p0 + step)) for p0 in range(0, c1 - c0, step)]
        list(pool.map(lambda pr: np.copyto(buf[pr[0]:pr[1]], src[c0 + pr[0]:c0 + pr[1]]), parts))
        with torch.cuda.stream(cs):
            dst[c0:c1].copy_(ring["bufs"][slot][: c1 - c0], non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(cs)
        ring["events"][slot] = ev
    torch.cuda.current_stream(dev).wait_stream(cs)
    return out


class HostPrefault:
    """Pageable result buffer whose pages are faulted in by a background thread
    while the device loop runs.  A fresh numpy result costs a kernel page fault
    plus a zeroed page per 4 KB on first touch -- at cfg2 the 2.3 GB W copied
    out at ~20 GB/s instead of the staging ring's ~31 -- and the host is idle
    during the loop.  One anonymous mapping of the largest possible result;
    ``advance(nbytes)`` lets the thread populate up to ``nbytes``
    (``madvise(MADV_POPULATE_WRITE)`` through ctypes, the GIL released; a
    strided touch where the kernel lacks it); ``array(shape, dtype)`` is the
    contiguous numpy view of the start, the mapping its base."""

    _CHUNK = 64 << 20

    def __init__(self, max_bytes, threads=4):
        import ctypes
        import mmap
        import threading
        from concurrent.futures import ThreadPoolExecutor

        self.size = max(int(max_bytes), mmap.PAGESIZE)
        self.mm = mmap.mmap(-1, self.size, flags=mmap.MAP_PRIVATE | mmap.MAP_ANONYMOUS)
        self.u8 = np.frombuffer(self.mm, dtype=np.uint8)
        self.addr = self.u8.ctypes.data
        self.libc = ctypes.CDLL(None, use_errno=True)
        self.libc.madvise.argtypes = [ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int]
        self.populate = True
        self.threads = threads
        self.pool = ThreadPoolExecutor(threads)
        self.target = self.done = 0
        self.stop = False
        self.cv = threading.Condition()
        self.thread = threading.Thread(target=self._run, daemon=True)
        self.thread.start()

    def advance(self, nbytes):
        with self.cv:
            self.target = max(self.target, min(self.size, int(nbytes)))
            self.cv.notify()

    def _touch(self, a, b):
        if self.populate and self.libc.madvise(self.addr + a, b - a, 23) == 0:  # MADV_POPULATE_WRITE
            return
        self.populate = False
        self.u8[a:b:4096] = 0

    def _run(self):
        pg = 4096
        while True:
            with self.cv:
                while not self.stop and self.done >= self.target:
                    self.cv.wait()
                if self.stop:
                    return
                a, b = self.done, min(self.target, self.done + self._CHUNK)
            a0 = a - a % pg
            b1 = min(self.size, -(-b // pg) * pg)
            part = -(-(b1 - a0) // (self.threads * pg)) * pg
            list(self.pool.map(lambda q: self._touch(q, min(b1, q + part)), range(a0, b1, part)))
            with self.cv:
                self.done = b

    def close(self):
        with self.cv:
            self.stop = True
            self.cv.notify()
        self.thread.join()
        self.pool.shutdown(wait=True)

    def array(self, shape, dtype):
        """The result view (stops the populating thread)."""
        self.close()
        dt = np.dtype(dtype)
        count = int(np.prod(shape))
        if count * dt.itemsize > self.size:
            return np.empty(shape, dtype=dt)
        return np.frombuffer(self.mm, dtype=dt, count=count).reshape(shape)


def d2h_pageable(x, out=None):
    """Fresh (pageable) numpy copy of a contiguous device tensor: 32 MB chunks
    are DMA'd into the pinned staging ring and copied out by the host thread
    pool while the next chunks are in flight -- no page-locking of the
    result (a caller that keeps every result would otherwise pin gigabytes
    per call)."""
    dev = x.device
    dt = torch.empty(0, dtype=x.dtype).numpy().dtype
    if isinstance(out, HostPrefault):
        out = out.array(tuple(x.shape), dt)
    elif out is None:
        out = np.empty(tuple(x.shape), dtype=dt)
    nbytes = x.numel() * x.element_size()
    if nbytes == 0:
        return out
    src = x.reshape(-1).view(torch.uint8)
    dst = out.reshape(-1).view(np.uint8)
    ring = _stage_ring(dev)
    pool = _copy_pool()
    nthr = max(1, min(16, pool._max_workers))
    cs = ring["stream"]
    cs.wait_stream(torch.cuda.current_stream(dev))
    waiting = {}  # slot -> (c0, c1) copied into the slot, not yet copied out

    def drain(slot):
        c0, c1 = waiting.pop(slot)
        ring["events"][slot].synchronize()
        buf = ring["bufs"][slot].numpy()
        n = c1 - c0
        part = -(-n // nthr)
        list(pool.map(lambda q: np.copyto(dst[c0 + q:c0 + min(n, q + part)], buf[q:min(n, q + part)]),
                      range(0, n, part)))

    for i, c0 in enumerate(range(0, nbytes, _STAGE_BYTES)):
        c1 = min(nbytes, c0 + _STAGE_BYTES)
        slot = i % _STAGE_DEPTH
        if slot in waiting:
            drain(slot)
        elif ring["events"][slot] is not None:
            ring["events"][slot].synchronize()
        with torch.cuda.stream(cs):
            ring["bufs"][slot][: c1 - c0].copy_(src[c0:c1], non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(cs)
        ring["events"][slot] = ev
        waiting[slot] = (c0, c1)
    for slot in sorted(waiting, key=lambda sl: waiting[sl][0]):
        drain(slot)
    return out


def h2d_rows(arr, on_chunk, out=None, align=1):
    """Row-chunked device copy of a C-contiguous 2-D host array: after each
    chunk's copy is enqueued, ``on_chunk(r0, r1, event)`` is called so work
    on the rows that have landed can be enqueued behind ``event`` while the
    rest is in flight.  Returns the device tensor; the current stream waits
    for the whole copy at the end.  Chunks are ~32 MB rounded to a multiple
    of ``align`` rows -- the same boundaries for pinned and pageable input,
    so the work on them (and its rounding) does not depend on the host
    allocation.  Pageable rows are staged through the pinned 32 MB ring."""
    dev = device()
    rows, cols = arr.shape
    host = torch.from_numpy(arr)
    if out is None:
        out = torch.empty(arr.shape, dtype=host.dtype, device=dev)
    pinned = host.is_pinned()
    row_bytes = max(1, arr.strides[0])
    ring = _stage_ring(dev)
    cs = ring["stream"]
    cs.wait_stream(torch.cuda.current_stream(dev))
    sub = max(1, _STAGE_BYTES // row_bytes)       # rows per pinned staging buffer
    step = max(align, sub // align * align)       # rows per chunk handed to on_chunk
    pool = _copy_pool()
    nthr = max(1, min(16, pool._max_workers))
    i = 0
    for r0 in range(0, rows, step):
        r1 = min(rows, r0 + step)
        if pinned:
            with torch.cuda.stream(cs):
                out[r0:r1].copy_(host[r0:r1], non_blocking=True)
                ev = torch.cuda.Event()
                ev.record(cs)
        else:
            for s0 in range(r0, r1, sub):
                s1 = min(r1, s0 + sub)
                slot = i % _STAGE_DEPTH
                i += 1
                prev = ring["events"][slot]
                if prev is not None:
                    prev.synchronize()
                nb = (s1 - s0) * row_bytes
                buf = ring["bufs"][slot].numpy()[:nb]
                src = arr[s0:s1].reshape(-1).view(np.uint8)
                part = -(-nb // nthr)
                list(pool.map(lambda q: np.copyto(buf[q:q + part], src[q:q + part]), range(0, nb, part)))
                with torch.cuda.stream(cs):
                    out[s0:s1].view(-1).view(torch.uint8).copy_(ring["bufs"][slot][:nb], non_blocking=True)
                    ev = torch.cuda.Event()
                    ev.record(cs)
                ring["events"][slot] = ev
        on_chunk(r0, r1, ev)
    torch.cuda.current_stream(dev).wait_stream(cs)
    return out


def as_index(idx, kind):
    """Index vector -> int64 device tensor."""
    if isinstance(idx, torch.Tensor):
        return idx.to(device=device(), dtype=torch.int64)
    return torch.as_tensor(np.asarray(idx, dtype=np.int64)).to(device())


def host_empty(shape, dtype=torch.float64):
    """Pinned host buffer (fast DMA) as a torch tensor."""
    return torch.empty(shape, dtype=dtype, pin_memory=True)


def to_output(x, like, host_out=None):
    """Return device tensor ``x`` in the container kind of ``like``
    (``host_out``: a `HostPrefault` to copy a large numpy result into)."""
    kind = like.kind if isinstance(like, Matrix) else like
    if isinstance(x, Matrix):
        x = x.t if not x.colmajor else x.t.t()
    if kind == "torch_cuda":
        if host_out is not None:
            host_out.close()
        return x
    if x.numel() >= (1 << 20) and x.is_contiguous() and kind == "numpy":
        return d2h_pageable(x, out=host_out)
    if host_out is not None:
        host_out.close()
    if x.numel() >= (1 << 20):
        h = host_empty(tuple(x.shape), x.dtype)
        h.copy_(x, non_blocking=True)
        torch.cuda.current_stream().synchronize()
    else:
        h = x.cpu()
    if kind == "torch_cpu":
        return h
    return h.numpy()


def to_host_index(x, kind):
    if kind == "torch_cuda":
        return x
    h = x.cpu()
    return h if kind == "torch_cpu" else h.numpy().astype(np.intp, copy=False)


def dgemm(a, b, alpha=1.0, beta=0.0, cin=None, out=None, aidx=None, bidx=None, cidx=None):
    """C = alpha * a @ b + beta * cin on the DMMA kernel.  a: Matrix (any
    layout), b: row-major Matrix; returns a row-major (M x N) torch tensor."""
    M, K = a.shape
    if aidx is not None:
        M = aidx.numel()
    N = b.cols
    if b.colmajor:
        b = b.row_major()
    if out is None:
        out = torch.empty((M, N), dtype=torch.float64, device=device())
    if cin is not None and cin.colmajor:
        cin = cin.row_major()
    _lib.call(
        "rs_dgemm", M, N, K, float(alpha), a.ptr, a.ld, int(a.colmajor),
        aidx.data_ptr() if aidx is not None else None,
        b.ptr, b.ld, bidx.data_ptr() if bidx is not None else None,
        float(beta), cin.ptr if cin is not None else None, cin.ld if cin is not None else 0,
        cidx.data_ptr() if cidx is not None else None,
        out.data_ptr(), out.stride(0) if out.dim() == 2 else N, workspace().data_ptr(),
        stream_handle(),
    )
    return out


def sketch(a, omega):
    """Y = a @ omega with omega a host (n x ell) float64 array (host-RNG draw)."""
    om = torch.as_tensor(np.ascontiguousarray(omega, dtype=np.float64)).to(device())
    return sketch_dev(a, om)


# ------------------------------------------------------------ device RNG ----
_rng_ws = {}


def _rng_workspace(n):
    need = _lib.load().rs_gaussian_workspace_bytes(n)
    dev = device()
    ws = _rng_ws.get(dev.index)
    if ws is None or ws.numel() < need:
        ws = torch.empty(int(need * 1.25) + 4096, dtype=torch.uint8, device=dev)
        _rng_ws[dev.index] = ws
    return ws


def host_rng():
    """RSKEL_HOST_RNG=1 draws Omega with numpy on the host (the reference's
    own generator) and copies it in, instead of the device draw."""
    import os
    return os.environ.get("RSKEL_HOST_RNG", "0") == "1"


def gaussian(stream, n, ell, unit=False, out=None, status=None):
    """(n, ell) standard normals of numpy's Generator(Philox(key=[seed, stream]))
    drawn on the device, divided by sqrt(ell) unless ``unit`` -- bit-identical
    to `make_gaussian` on the host (rs_gaussian).  ``stream`` is an RngStream.

    With ``status`` (a 1-element int32 device tensor) the launch is fully
    asynchronous and the caller checks ``status`` later; otherwise a nonzero
    status (a ziggurat chain longer than the parallel resolver supports, never
    observed) is repaired at once by the host draw."""
    dev = device()
    if out is None:
        out = torch.empty((n, ell), dtype=torch.float64, device=dev)
    N = n * ell
    if N == 0:
        return out
    ws = _rng_workspace(N)
    check = status is None
    if check:
        status = torch.empty(1, dtype=torch.int32, device=dev)
    scale = 1.0 if unit else float(np.sqrt(ell))
    k0, k1 = stream.philox_key()
    _lib.call("rs_gaussian", k0, k1, N, scale, out.data_ptr(),
              ws.data_ptr(), ws.numel(), status.data_ptr(), stream_handle())
    if check and int(status.item()) != 0:
        out.copy_(torch.as_tensor(host_gaussian(stream, n, ell, unit)))
    return out


def host_gaussian(stream, n, ell, unit=False):
    h = stream.generator().standard_normal((n, ell))
    if not unit:
        h /= np.sqrt(ell)
    return h


def omega_dense(spec, rng):
    """The (n x ell) embedding of ``spec`` from ``rng`` as a device tensor (any
    kind; Gaussian drawn on the device unless RSKEL_HOST_RNG=1)."""
    n, ell = spec.n, spec.ell
    if spec.kind != "gaussian":
        from .sketching import make_sketch

        return make_sketch(spec, rng).device_dense()
    unit = spec.scale != "inv_sqrt_ell"
    if host_rng():
        return torch.as_tensor(host_gaussian(rng, n, ell, unit)).to(device())
    return gaussian(rng, n, ell, unit=unit)


def sketch_omega(a, spec, rng):
    """Y = a @ Omega for the Gaussian embedding ``spec`` (n x ell) drawn from
    ``rng``: the device draw by default, the host draw under RSKEL_HOST_RNG=1.
    Same Omega bit for bit either way."""
    n, ell = spec.n, spec.ell
    if spec.kind != "gaussian":  # SRTT: dense on the device; sparse sign: SpMM
        from .sketching import make_sketch

        op = make_sketch(spec, rng)
        if spec.kind == "sparsesign":
            return sparse_sign_apply(a, op.idx, op.signs, op.ell, op.scale)
        return sketch_dev(a, op.device_dense())
    unit = spec.scale != "inv_sqrt_ell"
    if host_rng():
        om = torch.as_tensor(host_gaussian(rng, n, ell, unit)).to(device())
    else:
        om = gaussian(rng, n, ell, unit=unit)
    return sketch_dev(a, om)


def srtt_apply(a, perm, signs, cols, scale, out=None):
    """Y = a @ Omega for an SRTT Omega given by (perm, signs, cols, scale) as a fast
    transform (`rs_srtt_apply`: per-row DCT-II through one real FFT, O(m n log n))."""
    m, n = a.shape
    dev = device()
    ell = len(cols)
    perm, cols = np.asarray(perm), np.asarray(cols)
    for name, ix in (("perm", perm), ("cols", cols)):  # numpy's fancy indexing would raise the same
        if ix.size and (ix.min() < -n or ix.max() >= n):
            raise IndexError(f"SRTT {name} index out of bounds for size {n}")
    perm, cols = np.where(perm < 0, perm + n, perm), np.where(cols < 0, cols + n, cols)
    if len(perm) != n or len(np.asarray(signs)) != n:
        raise DimensionError(f"SRTT operator of size {len(perm)} does not match {n} columns")
    perm_d = torch.as_tensor(np.ascontiguousarray(perm, dtype=np.int64)).to(dev)
    sg_d = torch.as_tensor(np.ascontiguousarray(signs, dtype=np.float64)).to(dev)
    cols_d = torch.as_tensor(np.ascontiguousarray(cols, dtype=np.int64)).to(dev)
    lib = _lib.load()
    nbytes = min(int(lib.rs_srtt_workspace_bytes(m, n)), max(256 << 20, int(lib.rs_srtt_workspace_bytes(1, n))))
    ws = torch.empty(max(1, nbytes), dtype=torch.uint8, device=dev)
    y = out if out is not None else torch.empty((m, ell), dtype=torch.float64, device=dev)
    _lib.call("rs_srtt_apply", m, n, ell, a.ptr, a.ld, int(a.colmajor), perm_d.data_ptr(), sg_d.data_ptr(),
              cols_d.data_ptr(), float(scale), y.data_ptr(), y.stride(0), ws.data_ptr(), nbytes, stream_handle())
    return y


def sparse_sign_apply(a, idx, signs, ell, scale, out=None):
    """Y = a @ Omega for a sparse-sign Omega given by its (n x zeta) index and
    sign arrays, without forming Omega (`rs_sparse_sign_apply`; bitwise the
    reference's scipy SpMM).  ``out``: an (m x ell) row-major fp64 device tensor."""
    m, n = a.shape
    dev = device()
    idx_d = torch.as_tensor(np.ascontiguousarray(idx, dtype=np.int64)).to(dev)
    sg_d = torch.as_tensor(np.ascontiguousarray(signs, dtype=np.float64)).to(dev)
    zeta = idx_d.shape[1]
    plan = torch.empty(max(1, int(_lib.load().rs_sparse_sign_plan_bytes(n, ell))), dtype=torch.uint8, device=dev)
    bad = torch.zeros(1, dtype=torch.int32, device=dev)
    y = out if out is not None else torch.empty((m, ell), dtype=torch.float64, device=dev)
    _lib.call("rs_sparse_sign_apply", m, n, ell, zeta, a.ptr, a.ld, int(a.colmajor), idx_d.data_ptr(),
              sg_d.data_ptr(), float(scale), y.data_ptr(), y.stride(0), plan.data_ptr(), bad.data_ptr(),
              stream_handle())
    return y


def sketch_dev(a, om):
    """Y = a @ om with om a row-major (n x ell) device tensor."""
    m, n = a.shape
    ell = om.shape[1]
    y = torch.empty((m, ell), dtype=torch.float64, device=device())
    _lib.call("rs_sketch_gemm", m, n, ell, a.ptr, a.ld, int(a.colmajor), om.data_ptr(),
              max(ell, 1), y.data_ptr(), max(ell, 1), workspace().data_ptr(), stream_handle())
    return y
