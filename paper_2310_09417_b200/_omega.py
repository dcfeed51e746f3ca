"""Host Gaussian-block pipeline for the adaptive loop.

Block t of the adaptive loop draws Omega_t from ``rng.child(t)`` with the
per-block Gaussian normalisation (`skeleton.py:286-295`, variance 1/b).  The
blocks are independent Philox streams, so they are drawn ahead of use on a
thread pool (numpy releases the GIL inside ``standard_normal``), straight into
pinned host buffers, and copied to the device asynchronously on the compute
stream.  The bits are exactly the reference's: same generator, same C-order
fill, same in-place ``/= sqrt(b)``.
"""

import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import torch

from . import _device

_POOL = None


def _pool():
    global _POOL
    if _POOL is None:
        _POOL = ThreadPoolExecutor(max_workers=max(1, os.cpu_count() or 1),
                                   thread_name_prefix="rskel-omega")
    return _POOL


def workers():
    return _pool()._max_workers


def draw_block_pinned(n, ell, stream, unit_scale):
    """Pinned (n, ell) host tensor holding ``stream``'s standard normals
    (scaled by 1/sqrt(ell) unless unit_scale)."""
    h = torch.empty((n, ell), dtype=torch.float64, pin_memory=True)
    buf = h.numpy()
    stream.generator().standard_normal(out=buf)
    if not unit_scale:
        buf /= np.sqrt(ell)
    return h


class BlockOmegaSource:
    """Omega_t (n x b), t = 0, 1, ..., drawn ``depth`` blocks ahead."""

    def __init__(self, n, b, rng, unit_scale=False, depth=None):
        self.n, self.b, self.rng, self.unit = n, b, rng, unit_scale
        self.depth = depth or 2 * workers()
        self._futs = {}
        self._next = 0

    def _submit_upto(self, t_end):
        while self._next < t_end:
            t = self._next
            self._futs[t] = _pool().submit(draw_block_pinned, self.n, self.b, self.rng.child(t), self.unit)
            self._next += 1

    def host(self, t):
        self._submit_upto(t + self.depth)
        fut = self._futs.pop(t, None)
        if fut is None:  # out-of-order request
            return draw_block_pinned(self.n, self.b, self.rng.child(t), self.unit)
        return fut.result()

    def device(self, t, out=None):
        h = self.host(t)
        if out is None:
            out = torch.empty((self.n, self.b), dtype=torch.float64, device=_device.device())
        out.copy_(h, non_blocking=True)
        return out

    def close(self):
        for f in self._futs.values():
            f.cancel()
        self._futs.clear()
