"""Seeded embeddings and their application on the B200.

Every embedding is defined by numpy's Philox4x64 generator keyed by a
``(seed, stream)`` pair exactly as in the reference (`sketching.py:41-72`),
so the operator bits are the reference's:

* Gaussian (`sketching.py:191-204`): drawn on the device by `rs_gaussian`
  (bit-identical to numpy's ziggurat) on the skeleton paths; `make_gaussian`
  keeps the host draw.
* SRTT (`sketching.py:134-157,207-216`) and sparse sign
  (`sketching.py:160-187,219-235`): the operator parameters (permutation,
  signs, sampled columns / row supports) come from the same numpy calls as
  the reference; the dense n x ell embedding is formed on the device
  (`rs_srtt_dense`, `rs_sparse_sign_dense`).

Applying any embedding (``a @ Omega``) runs on the DMMA GEMM kernel of
librskel.so (`rs_sketch_gemm`).
"""

from dataclasses import dataclass, replace
from functools import lru_cache

import numpy as np

from . import _device
from .errors import DimensionError

__all__ = [
    "SketchSpec",
    "RngStream",
    "GaussianSketch",
    "SrttSketch",
    "SparseSignSketch",
    "make_gaussian",
    "make_srtt",
    "make_sparse_sign",
    "make_sketch",
    "apply_sketch",
]

KINDS = ("gaussian", "srtt", "sparsesign")
SCALES = ("unit", "inv_sqrt_ell")

_M64 = 0xFFFFFFFFFFFFFFFF


def _splitmix64(z):
    """SplitMix64 output function (Steele, Lea & Flood 2014); the stream
    derivation of the reference `sketching.py:47-52`."""
    z = (z + 0x9E3779B97F4A7C15) & _M64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _M64
    return z ^ (z >> 31)


@lru_cache(maxsize=4096)
def _philox_key(seed, stream):
    k = np.random.Philox(key=[seed, stream]).state["state"]["key"]
    return int(k[0]), int(k[1])


@dataclass(frozen=True)
class RngStream:
    """Reproducible splittable stream: Philox4x64 keyed by ``[seed, stream]``
    (reference `sketching.py:55-72`)."""

    seed: int
    stream: int = 0

    def generator(self):
        return np.random.Generator(np.random.Philox(key=[self.seed & _M64, self.stream & _M64]))

    def philox_key(self):
        """The two key words numpy's Philox really runs with for
        ``key=[seed, stream]``: numpy converts the list with np.asarray, which
        goes through float64 when one word is >= 2**63 and the other is not,
        rounding that word.  The device draw must use the same words."""
        return _philox_key(self.seed & _M64, self.stream & _M64)

    def child(self, i):
        return RngStream(self.seed, _splitmix64((self.stream & _M64) ^ _splitmix64(i & _M64)))


@dataclass(frozen=True)
class SketchSpec:
    """Embedding description Omega in R^{n x ell} (reference `sketching.py:75-109`)."""

    kind: str
    n: int
    ell: int
    scale: str = "inv_sqrt_ell"
    zeta: int = 8
    seed: int = 0

    def __post_init__(self):
        if self.kind not in KINDS:
            raise ValueError(f"unknown sketch kind {self.kind!r}; expected one of {KINDS}")
        if self.scale not in SCALES:
            raise ValueError(f"unknown scale {self.scale!r}; expected one of {SCALES}")
        if not 1 <= self.ell <= self.n:
            raise DimensionError(
                f"embedding dimension must satisfy 1 <= ell <= n, got ell={self.ell}, n={self.n}"
            )
        if self.kind == "sparsesign" and not 2 <= self.zeta <= self.ell:
            raise DimensionError(
                f"sparse sign needs 2 <= zeta <= ell, got zeta={self.zeta}, ell={self.ell}"
            )

    def with_dims(self, n, ell):
        return replace(self, n=n, ell=ell)


def make_gaussian(spec, rng):
    """Host draw of the (n, ell) Gaussian embedding, C-order fill, then
    ``/= sqrt(ell)`` for the 'inv_sqrt_ell' scale (reference `sketching.py:191-204`)."""
    if spec.kind != "gaussian":
        raise ValueError(f"spec kind is {spec.kind!r}, expected 'gaussian'")
    omega = rng.generator().standard_normal((spec.n, spec.ell))
    if spec.scale == "inv_sqrt_ell":
        omega /= np.sqrt(spec.ell)
    return omega


class GaussianSketch:
    """Dense Gaussian embedding; ``apply`` runs the device sketch GEMM."""

    def __init__(self, omega):
        self.omega = omega

    @property
    def shape(self):
        return self.omega.shape

    def apply(self, a):
        a = _device.as_matrix(a)
        if a.cols != self.omega.shape[0]:
            raise DimensionError(
                f"operator ambient dimension {self.omega.shape[0]} does not match {a.shape}"
            )
        y = _device.sketch(a, self.omega)
        return _device.to_output(y, a)

    def to_dense(self):
        return self.omega


def _apply_dense(op, a):
    A = _device.as_matrix(a)
    n = op.shape[0]
    if A.cols != n:
        raise DimensionError(f"operator ambient dimension {n} does not match {A.shape}")
    return _device.to_output(_device.sketch_dev(A, op.device_dense()), A)


SRTT_FFT_MIN_ELL = 512  # sampled columns from which the FFT form beats the dense product (~450 at 20000^2)


class SrttSketch:
    """Subsampled randomized trigonometric transform (reference
    `sketching.py:134-157`): ``y = scale * (DCT-II(x[perm]) * signs)[cols]``."""

    def __init__(self, perm, signs, cols, scale):
        self.perm, self.signs, self.cols, self.scale = perm, signs, cols, scale

    @property
    def shape(self):
        return (self.perm.shape[0], self.cols.shape[0])

    def device_dense(self):
        import torch

        from . import _lib

        n, ell = self.shape
        dev = _device.device()
        out = torch.empty((n, ell), dtype=torch.float64, device=dev)
        perm = torch.as_tensor(np.asarray(self.perm, dtype=np.int64)).to(dev)
        cols = torch.as_tensor(np.asarray(self.cols, dtype=np.int64)).to(dev)
        signs = torch.as_tensor(np.asarray(self.signs, dtype=np.float64)).to(dev)
        _lib.call("rs_srtt_dense", n, ell, perm.data_ptr(), signs.data_ptr(), cols.data_ptr(), float(self.scale),
                  out.data_ptr(), ell, _device.stream_handle())
        return out

    def apply(self, a):
        """``a @ Omega``: for ell >= SRTT_FFT_MIN_ELL as the reference computes it, a
        length-n DCT per row (`rs_srtt_apply`, O(m n log n)); below that the dense
        embedding on the sketch engine is the cheaper pass over A."""
        A = _device.as_matrix(a)
        if A.cols != self.shape[0]:
            raise DimensionError(f"operator ambient dimension {self.shape[0]} does not match {A.shape}")
        if self.shape[1] >= SRTT_FFT_MIN_ELL:
            return _device.to_output(_device.srtt_apply(A, self.perm, self.signs, self.cols, self.scale), A)
        return _apply_dense(self, A)

    def to_dense(self):
        return self.device_dense().cpu().numpy()


class SparseSignSketch:
    """Sparse-sign embedding, ``zeta`` (index, sign) pairs per row scaled by
    ``scale`` (reference `sketching.py:160-187`)."""

    def __init__(self, idx, signs, ell, scale):
        self.idx, self.signs, self.ell, self.scale = idx, signs, ell, scale
        self._exact = None

    @property
    def shape(self):
        return (self.idx.shape[0], self.ell)

    def spmm_exact(self):
        """True when the operator is one the SpMM reproduces bitwise: signs of
        +-1 and no index repeated within a row (every `make_sparse_sign` draw).
        Hand-built operators outside that use the dense device form."""
        if self._exact is None:
            idx = np.asarray(self.idx)
            srt = np.sort(idx, axis=1)
            self._exact = bool(np.all(np.abs(np.asarray(self.signs)) == 1.0)
                               and np.all(srt[:, 1:] != srt[:, :-1])
                               and idx.min(initial=0) >= 0 and idx.max(initial=0) < self.ell)
        return self._exact

    def device_dense(self):
        import torch

        from . import _lib

        n, zeta = self.idx.shape
        dev = _device.device()
        out = torch.empty((n, self.ell), dtype=torch.float64, device=dev)
        idx = torch.as_tensor(np.ascontiguousarray(self.idx, dtype=np.int64)).to(dev)
        signs = torch.as_tensor(np.ascontiguousarray(self.signs, dtype=np.float64)).to(dev)
        _lib.call("rs_sparse_sign_dense", n, self.ell, zeta, idx.data_ptr(), signs.data_ptr(), float(self.scale),
                  out.data_ptr(), self.ell, _device.stream_handle())
        return out

    def apply(self, a):
        """``a @ Omega`` as an SpMM over the (index, sign) pairs, bitwise the
        reference's `(csr.T @ a.T).T` (`sketching.py:176-185`)."""
        if not self.spmm_exact():
            return _apply_dense(self, a)
        A = _device.as_matrix(a)
        if A.cols != self.shape[0]:
            raise DimensionError(f"operator ambient dimension {self.shape[0]} does not match {A.shape}")
        return _device.to_output(_device.sparse_sign_apply(A, self.idx, self.signs, self.ell, self.scale), A)

    def to_dense(self):
        return self.device_dense().cpu().numpy()


def make_srtt(spec, rng):
    """SRTT operator: permutation, signs, sampled columns from the stream in
    the reference's order (`sketching.py:207-216`)."""
    if spec.kind != "srtt":
        raise ValueError(f"spec kind is {spec.kind!r}, expected 'srtt'")
    g = rng.generator()
    perm = g.permutation(spec.n)
    signs = g.integers(0, 2, size=spec.n) * 2.0 - 1.0
    cols = g.choice(spec.n, size=spec.ell, replace=False)
    return SrttSketch(perm.astype(np.intp), signs, cols.astype(np.intp), np.sqrt(spec.n / spec.ell))


def make_sparse_sign(spec, rng):
    """Sparse-sign operator: a uniform zeta-subset of the ell columns per row
    (ranks of i.i.d. uniforms) and Rademacher signs scaled by 1/sqrt(zeta)
    (`sketching.py:219-235`)."""
    if spec.kind != "sparsesign":
        raise ValueError(f"spec kind is {spec.kind!r}, expected 'sparsesign'")
    g = rng.generator()
    u = g.random((spec.n, spec.ell))
    idx = np.argsort(u, axis=1)[:, : spec.zeta]
    signs = g.integers(0, 2, size=(spec.n, spec.zeta)) * 2.0 - 1.0
    return SparseSignSketch(np.ascontiguousarray(idx, dtype=np.intp), signs, spec.ell, 1.0 / np.sqrt(spec.zeta))


def make_sketch(spec, rng):
    """Construct the operator described by ``spec`` (reference `sketching.py:238-244`)."""
    if spec.kind == "gaussian":
        return GaussianSketch(make_gaussian(spec, rng))
    if spec.kind == "srtt":
        return make_srtt(spec, rng)
    return make_sparse_sign(spec, rng)


def apply_sketch(a, op, side="right"):
    """``a @ Omega`` (side='right') or ``a.T @ Gamma`` ('transposed_right') on
    the device (reference `sketching.py:247-273`)."""
    a = _device.as_matrix(a)
    if side not in ("right", "transposed_right"):
        raise ValueError(f"side must be 'right' or 'transposed_right', got {side!r}")
    target = a if side == "right" else a.T
    if isinstance(op, (SrttSketch, SparseSignSketch)):
        if target.cols != op.shape[0]:
            raise DimensionError(f"operator ambient dimension {op.shape[0]} does not match {target.shape}")
        if isinstance(op, SparseSignSketch) and op.spmm_exact():
            return _device.to_output(_device.sparse_sign_apply(target, op.idx, op.signs, op.ell, op.scale), a)
        if isinstance(op, SrttSketch) and op.shape[1] >= SRTT_FFT_MIN_ELL:
            return _device.to_output(_device.srtt_apply(target, op.perm, op.signs, op.cols, op.scale), a)
        return _device.to_output(_device.sketch_dev(target, op.device_dense()), a)
    omega = op if isinstance(op, np.ndarray) else getattr(op, "omega", None)
    if omega is None:
        raise TypeError("op must be a sketch operator or a dense embedding matrix")
    omega = np.asarray(omega, dtype=np.float64)
    if target.cols != omega.shape[0]:
        if isinstance(op, np.ndarray):
            raise DimensionError(f"dimension mismatch: {target.shape} x {omega.shape}")
        raise DimensionError(
            f"operator ambient dimension {omega.shape[0]} does not match {target.shape}"
        )
    y = _device.sketch(target, omega)
    return _device.to_output(y, a)
