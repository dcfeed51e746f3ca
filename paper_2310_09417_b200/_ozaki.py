"""Host side of the tensor-core sketch (csrc/ozaki.cu): digit planes of the
sketched matrix and of each Omega block, and the plane GEMM.

The adaptive loop multiplies the same A by a fresh Gaussian block every
iteration (`skeleton.py:437-441`).  A is therefore cut into int8 digit
planes once per call (`Planes.of_matrix`), Omega_t per block
(`Planes.of_omega`), and every block's sketch Y_t = A Omega_t runs as exact
int32 plane products on the tcgen05 int8 pipe (`sketch`).  The summation
order depends on K alone, as for the DMMA GEMM, so a row of Y has the same
bits on one GPU, on any rank of the column-sharded loop, and for device or
host input.

Engine selection (`set_sketch_engine`): "ozaki" (default) or "dmma" (the
fp64 DMMA GEMM of gemm_f64.cu) -- the latter keeps the r01 arithmetic for
comparisons.
"""

import torch

from . import _device, _lib

A_PLANES = {torch.float64: 8, torch.float32: 4}  # 7-bit digits per entry: 56 / 28 bits
OMEGA_PLANES = 8
_TILE_A, _TILE_B = 128, 64
_ENGINE = {"sketch": "ozaki"}


def set_sketch_engine(name):
    """Choose the arithmetic of the adaptive loop's sketch GEMM: "ozaki"
    (int8 tensor cores, default) or "dmma" (fp64 DMMA)."""
    if name not in ("ozaki", "dmma"):
        raise ValueError(f"unknown sketch engine {name!r}")
    _ENGINE["sketch"] = name


def sketch_engine():
    return _ENGINE["sketch"]


class Planes:
    """Digit planes + per-(row, K-chunk) exponents of a rows x K operand."""

    def __init__(self, rows, K, S, tile_rows, dev):
        lib = _lib.load()
        self.rows, self.K, self.S, self.tile_rows = rows, K, S, tile_rows
        self.kc = lib.rs_oz_chunk(K)
        self.nch = max(1, -(-K // self.kc))
        self.dig = torch.empty(max(1, lib.rs_oz_digits_bytes(rows, K, S, tile_rows)), dtype=torch.int8, device=dev)
        self.expo = torch.empty(max(1, rows * self.nch), dtype=torch.int32, device=dev)
        self.nonfinite = torch.zeros(1, dtype=torch.int32, device=dev)

    def fill(self, ptr, fp32, ld, colmajor, k0=0, k1=None, ws=None):
        """Planes of columns [k0, k1) of the operand at ``ptr`` (element (i, k)
        at ptr[i*ld + k], or ptr[k*ld + i] when ``colmajor``)."""
        k1 = self.K if k1 is None else k1
        _lib.call("rs_oz_slice", ptr, int(fp32), ld, int(colmajor), self.rows, self.K, k0, k1, self.kc, self.S,
                  self.tile_rows, self.dig.data_ptr(), self.expo.data_ptr(), self.nonfinite.data_ptr(),
                  (ws if ws is not None else _device.workspace()).data_ptr(), _device.stream_handle())
        return self

    def fill_rows(self, ptr, fp32, ld, r0, r1):
        """Planes of rows [r0, r1) (r0 a multiple of the tile height) of a
        row-major operand whose row r0 starts at ``ptr``."""
        assert r0 % self.tile_rows == 0
        lib = _lib.load()
        dig_off = lib.rs_oz_digits_bytes(r0, self.K, self.S, self.tile_rows)
        _lib.call("rs_oz_slice", ptr, int(fp32), ld, 0, r1 - r0, self.K, 0, self.K, self.kc, self.S,
                  self.tile_rows, self.dig.data_ptr() + dig_off, self.expo.data_ptr() + 4 * r0 * self.nch,
                  self.nonfinite.data_ptr(), _device.workspace().data_ptr(), _device.stream_handle())
        return self

    @classmethod
    def of_matrix(cls, a):
        """Planes of the candidate matrix (a device Matrix); fp32 input
        (``a.src32``) is sliced from its fp32 values: 4 planes = 28 bits, 4
        bytes per entry instead of 8."""
        src = a.src32
        if src is not None:
            return cls(a.rows, a.cols, A_PLANES[torch.float32], _TILE_A, a.t.device).fill(
                src.t.data_ptr() + 4 * src.off, True, src.ld, src.colmajor)
        return cls(a.rows, a.cols, A_PLANES[torch.float64], _TILE_A, a.t.device).fill(a.ptr, False, a.ld, a.colmajor)

    @classmethod
    def of_omega(cls, om, out=None, ws=None):
        """Planes of Omega (n x N row-major fp64): rows = its N columns."""
        n, N = om.shape
        p = out if out is not None else cls(N, n, OMEGA_PLANES, _TILE_B, om.device)
        return p.fill(om.data_ptr(), False, om.stride(0), True, ws=ws)


def sketch(ap, bp, y_ptr, ldy, ws=None):
    """Y (M x N, row-major at y_ptr) = A Omega from their planes."""
    _lib.call("rs_oz_gemm", ap.rows, bp.rows, ap.K, ap.kc, 0, 1.0, ap.dig.data_ptr(), ap.expo.data_ptr(), ap.S,
              bp.dig.data_ptr(), bp.expo.data_ptr(), bp.S, 0.0, None, 0, y_ptr, ldy,
              (ws if ws is not None else _device.workspace()).data_ptr(), _device.stream_handle())
