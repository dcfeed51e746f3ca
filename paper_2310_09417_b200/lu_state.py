"""LU-form adaptive state -- the resumable API of the reference
(`skeleton.py:152-197,286-388`): BlockedLUState, adaptive_init,
adaptive_step, interpolation_matrix.

`rand_lupp_adaptive` itself runs on the T-form engine (`skeleton.py` here);
these entry points keep the reference's explicit (L1, L2, U1, ysofar) state
for callers that drive the loop themselves.  Every product, solve and
factorisation runs on the device kernels (`dense.py` here).
"""

import math
from dataclasses import dataclass, replace

import numpy as np
import torch

from . import _device, dense
from .errors import DimensionError
from .sketching import make_sketch

__all__ = ["BlockedLUState", "adaptive_init", "adaptive_step", "interpolation_matrix", "ResidualEstimates",
           "draw_residual_sample", "residual_ur_estimates"]

_RESIDUAL_STREAM = 1 << 40  # reference `skeleton.py:75`


@dataclass
class BlockedLUState:
    """``ysofar[perm] = [[L1], [L2]] @ U1`` with L1 unit lower triangular
    (reference `skeleton.py:152-173`).  Arrays are numpy for numpy inputs and
    CUDA tensors for CUDA-tensor inputs."""

    t: int
    b: int
    m: int
    L1: object
    L2: object
    U1: object
    perm: object
    ysofar: object
    rng: object

    @property
    def rank(self):
        return self.U1.shape[0]


def _block_spec(spec, n, ell):
    """Per-block spec: Gaussian blocks use variance 1/ell (`skeleton.py:276-290`)."""
    from dataclasses import replace

    kwargs = {"n": n, "ell": ell}
    if spec.kind == "gaussian":
        kwargs["scale"] = "inv_sqrt_ell"
    if spec.kind == "sparsesign" and spec.zeta > ell:
        kwargs["zeta"] = ell
    return replace(spec, **kwargs)


def _draw_block(A, spec, stream, b):
    """``a @ Omega`` for one block (`skeleton.py:293-295`) -> device tensor (m x b)."""
    return _device.sketch_omega(A, _block_spec(spec, A.cols, b), stream)


def _kind_out(x, kind):
    if kind == "torch_cuda":
        return x
    return _device.to_output(x.contiguous(), kind)


def _dev(x):
    if isinstance(x, torch.Tensor):
        return x.to(device=_device.device(), dtype=torch.float64)
    return torch.as_tensor(np.ascontiguousarray(x, dtype=np.float64)).to(_device.device())


def _devi(x):
    if isinstance(x, torch.Tensor):
        return x.to(device=_device.device(), dtype=torch.int64)
    return torch.as_tensor(np.asarray(x, dtype=np.int64)).to(_device.device())


def adaptive_init(a, b, spec, rng):
    """First block: sketch and factor (reference `skeleton.py:298-314`)."""
    m, n = _device.shape_of(a)
    if not 1 <= b <= min(m, n):
        raise DimensionError(f"block size must be in [1, {min(m, n)}], got {b}")
    A = _device.as_matrix(a)
    y = _draw_block(A, spec, rng.child(0), b)
    f = dense.lupp(y)  # CUDA tensor in -> CUDA tensors out
    kind = A.kind
    return BlockedLUState(
        t=1, b=b, m=m,
        L1=_kind_out(f.L[:b].clone(), kind), L2=_kind_out(f.L[b:].clone(), kind),
        U1=_kind_out(f.U, kind), perm=_device.to_host_index(f.perm, kind),
        ysofar=_kind_out(y, kind), rng=rng,
    )


def _schur(L1, L2, perm, y):
    """(U2, S) of a fresh block (reference `skeleton.py:317-323`)."""
    k = L1.shape[0]
    py = dense._gather_rows(dense._mat(y.contiguous()), perm).tensor()
    u2 = dense.triangular_solve(L1, py[:k], side="left", uplo="lower", unit_diagonal=True)
    s = torch.empty((py.shape[0] - k, py.shape[1]), dtype=torch.float64, device=py.device)
    dense._gemm(dense._mat(s), dense._mat(L2.contiguous()), dense._mat(u2.contiguous()), alpha=-1.0,
                beta=1.0, Cin=dense._mat(py[k:].contiguous()))
    return u2, s


def adaptive_step(state, a, spec, rng=None):
    """One estimate + absorb step (reference `skeleton.py:354-388`).
    Returns ``(e_schur, new_state)``."""
    m, n = _device.shape_of(a)
    k = state.rank
    if k + state.b > min(m, n):
        raise DimensionError(
            f"cannot extend rank {k} by block {state.b} beyond min(m, n) = {min(m, n)}"
        )
    A = _device.as_matrix(a)
    kind = A.kind
    stream = (rng or state.rng).child(state.t)
    y = _draw_block(A, spec, stream, state.b)
    L1, L2, U1 = _dev(state.L1), _dev(state.L2), _dev(state.U1)
    perm = _devi(state.perm)
    u2, s = _schur(L1, L2, perm, y)
    e_schur = dense.frobenius_norm(s)
    sub = dense.lupp(s)
    b = state.b
    l2p = L2[sub.perm]
    L1n = torch.zeros((k + b, k + b), dtype=torch.float64, device=L1.device)
    L1n[:k, :k] = L1
    L1n[k:, :k] = l2p[:b]
    L1n[k:, k:] = sub.L[:b]
    L2n = torch.cat([l2p[b:], sub.L[b:]], dim=1)
    U1n = torch.zeros((k + b, k + b), dtype=torch.float64, device=L1.device)
    U1n[:k, :k] = U1
    U1n[:k, k:] = u2
    U1n[k:, k:] = sub.U
    pn = perm.clone()
    pn[k:] = perm[k:][sub.perm]
    ys = torch.cat([_dev(state.ysofar), y], dim=1)
    new = BlockedLUState(
        t=state.t + 1, b=b, m=state.m,
        L1=_kind_out(L1n, kind), L2=_kind_out(L2n.contiguous(), kind), U1=_kind_out(U1n, kind),
        perm=_device.to_host_index(pn, kind), ysofar=_kind_out(ys, kind), rng=state.rng,
    )
    return e_schur, new


def interpolation_matrix(state):
    """W with W[perm[:k]] = I and W[perm[k:]] = L2 L1^{-1} (reference `skeleton.py:192-197`)."""
    from . import _lib

    L1, L2 = _dev(state.L1), _dev(state.L2)
    k = L1.shape[0]
    t_block = dense.triangular_solve(L1, L2, side="right", uplo="lower", unit_diagonal=True)
    T = t_block if isinstance(t_block, torch.Tensor) and t_block.is_cuda else _dev(t_block)
    T = T.contiguous()
    perm = _devi(state.perm)
    m = perm.numel()
    W = torch.empty((m, k), dtype=torch.float64, device=T.device)
    _lib.call("rs_scatter_interp", T.data_ptr(), max(k, 1), perm.data_ptr(), m, k, W.data_ptr(),
              max(k, 1), _device.stream_handle())
    kind = "torch_cuda" if isinstance(state.L1, torch.Tensor) and state.L1.is_cuda else "numpy"
    return _kind_out(W, kind)


@dataclass
class ResidualEstimates:
    """Error proxies from the trailing p x p factor of a dedicated sample
    (reference `skeleton.py:142-149`)."""

    norm_ur: float
    max_ur: float
    est_norm: float
    est_max: float


def draw_residual_sample(a, p, spec, rng):
    """Dedicated sample ``a @ Omega_r`` (m x p) from ``rng.child(1 << 40)``,
    unit-variance Gaussian Omega_r drawn on the device (reference
    `skeleton.py:527-539`)."""
    m, n = _device.shape_of(a)
    A = _device.as_matrix(a)
    stream = rng.child(_RESIDUAL_STREAM)
    if spec.kind == "gaussian":
        sp = replace(spec, n=n, ell=p, scale="unit")
    else:  # `_sized_spec`: sparse-sign rows saturate at zeta = ell
        sp = replace(spec, n=n, ell=p, zeta=min(spec.zeta, p) if spec.kind == "sparsesign" else spec.zeta)
    y = _device.sketch_omega(A, sp, stream)
    return _kind_out(y, A.kind)


def residual_ur_estimates(state, a, p, spec, rng, sample_r=None):
    """Norms of the trailing p x p LU factor of a dedicated sample reduced
    against the state, scaled by ``(4 log k / k) sqrt(m - k)`` (reference
    `skeleton.py:463-524`)."""
    m, n = _device.shape_of(a)
    if not 1 <= p < state.b:
        raise DimensionError(f"oversample count must satisfy 1 <= p < b = {state.b}")
    k = state.rank
    if m - k < p:
        raise DimensionError(f"need at least p = {p} rows beyond rank {k}")
    if sample_r is None:
        y_r = _dev(draw_residual_sample(a, p, spec, rng))
    else:
        shp = tuple(sample_r.shape)
        if shp != (m, p):
            raise DimensionError(f"sample_r must have shape {(m, p)}, got {shp}")
        y_r = _dev(sample_r)
    L1, L2 = _dev(state.L1), _dev(state.L2)
    perm = _devi(state.perm)
    _, s_r = _schur(L1, L2, perm, y_r)
    _, U, _, nc = dense._lupp_partial_device(dense._mat(s_r.contiguous()))
    if nc == 0:
        norm_ur = max_ur = 0.0
    else:
        norm_ur = dense.frobenius_norm(U)
        max_ur = float(U.abs().max().item())
    factor = (4.0 * math.log(k) / k) * math.sqrt(m - k)
    if spec.kind != "gaussian":
        factor *= math.sqrt(p)
    return ResidualEstimates(norm_ur=norm_ur, max_ur=max_ur, est_norm=factor * norm_ur, est_max=factor * max_ur)
