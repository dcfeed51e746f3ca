"""Digit planes of the tensor-core sketch (`rs_oz_slice`) against a numpy restatement of the
Ozaki split, byte for byte: per (row, K-chunk) exponent e of the chunk maximum (frexp), y =
x 2^-e, then S signed 7-bit digits d_s = trunc(128 y_s), y_{s+1} = 128 y_s - d_s, stored in
the swizzled tile layout the MMA's shared-memory descriptors read."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

BK = 128


def _digits_numpy(x, kc, S):
    rows, K = x.shape
    nch = -(-K // kc)
    d = np.zeros((S, rows, K), dtype=np.int8)
    expo = np.zeros((rows, nch), dtype=np.int32)
    for c in range(nch):
        blk = x[:, c * kc:(c + 1) * kc]
        m = np.abs(blk).max(axis=1)
        _, e = np.frexp(m)
        e = np.where(m > 0, e, 0).astype(np.int32)
        expo[:, c] = e
        y = np.ldexp(blk, -e[:, None])
        for s in range(S):
            z = y * 128.0
            t = np.trunc(z)
            d[s, :, c * kc:(c + 1) * kc] = t.astype(np.int8)
            y = z - t
    return d, expo


def _decode(dig, rows, K, S, tile_rows):
    """The device's tile layout back to (S, rows, K) int8."""
    KB = -(-K // BK)
    tb = tile_rows * BK
    out = np.zeros((S, rows, K), dtype=np.int8)
    i = np.arange(rows)[:, None]
    k = np.arange(K)[None, :]
    tile, r, kb, c16, j = i // tile_rows, i % tile_rows, k // BK, (k % BK) // 16, k % 16
    for s in range(S):
        addr = ((tile * KB + kb) * S + s) * tb + (r >> 3) * 1024 + (r & 7) * 128 + ((c16 ^ (r & 7)) * 16) + j
        out[s] = dig[addr]
    return out


@pytest.mark.parametrize("rows,K,colmajor,fp32,tile_rows", [
    (200, 3000, False, False, 128), (64, 2500, True, False, 64), (130, 1030, False, True, 128),
    (37, 777, True, True, 64),
])
def test_planes_bytes_match_numpy(rows, K, colmajor, fp32, tile_rows):
    import torch

    from paper_2310_09417_b200 import _ozaki

    g = np.random.default_rng(rows + K)
    x = g.standard_normal((rows, K)) * np.exp2(g.integers(-60, 60, size=(rows, 1)))
    x[:, 5] = 0.0
    x[3, :] = 0.0                                  # an all-zero row
    x[7, :40] = np.exp2(g.integers(-1030, -1000, size=40)) * 1.5  # near-denormal chunk entries
    x[9, 11] = 2.0 ** 40                           # an exact power of two as a chunk max
    x[10, :] = -np.abs(x[10, :])                   # a negative row
    if fp32:
        x = np.clip(x, -1e30, 1e30).astype(np.float32).astype(np.float64)
    S = 4 if fp32 else 8
    kc = _ozaki._lib.load().rs_oz_chunk(K)
    src = np.asfortranarray(x) if colmajor else np.ascontiguousarray(x)
    t = torch.as_tensor(src.astype(np.float32) if fp32 else src).cuda()
    ld = rows if colmajor else K
    p = _ozaki.Planes(rows, K, S, tile_rows, t.device).fill(t.data_ptr(), fp32, ld, colmajor)
    torch.cuda.synchronize()
    want_d, want_e = _digits_numpy(x, kc, S)
    assert np.array_equal(p.expo.cpu().numpy().reshape(rows, -1), want_e)
    got = _decode(p.dig.cpu().numpy(), rows, K, S, tile_rows)
    assert np.array_equal(got, want_d)
