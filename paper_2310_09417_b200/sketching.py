"""Seeded Gaussian embeddings and their application on the B200.

Host-RNG contract (north star: "Omega supplied from the host RNG"): every
embedding is drawn on the host from numpy's Philox4x64 generator keyed by a
``(seed, stream)`` pair exactly as the reference does (`sketching.py:41-72`,
`sketching.py:191-204`), so the Omega bits are identical to the reference's.
Applying the embedding (``a @ Omega``) runs on the DMMA GEMM kernel of
librskel.so (`rs_sketch_gemm`).

Only the Gaussian distribution is on the accelerated path; SRTT and sparse
sign specs validate like the reference but ``make_sketch`` rejects them (they
are out of the north-star scope).
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
    "make_gaussian",
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


def make_sketch(spec, rng):
    """Construct the operator described by ``spec`` (Gaussian only here)."""
    if spec.kind == "gaussian":
        return GaussianSketch(make_gaussian(spec, rng))
    raise NotImplementedError(
        f"sketch kind {spec.kind!r} is outside the B200 hot path (Gaussian only)"
    )


def apply_sketch(a, op, side="right"):
    """``a @ Omega`` (side='right') or ``a.T @ Gamma`` ('transposed_right') on
    the device (reference `sketching.py:247-273`)."""
    a = _device.as_matrix(a)
    if side not in ("right", "transposed_right"):
        raise ValueError(f"side must be 'right' or 'transposed_right', got {side!r}")
    target = a if side == "right" else a.T
    omega = op if isinstance(op, np.ndarray) else getattr(op, "omega", None)
    if omega is None:
        raise NotImplementedError("only dense Gaussian embeddings are applied on the device")
    omega = np.asarray(omega, dtype=np.float64)
    if target.cols != omega.shape[0]:
        if isinstance(op, np.ndarray):
            raise DimensionError(f"dimension mismatch: {target.shape} x {omega.shape}")
        raise DimensionError(
            f"operator ambient dimension {omega.shape[0]} does not match {target.shape}"
        )
    y = _device.sketch(target, omega)
    return _device.to_output(y, a)
