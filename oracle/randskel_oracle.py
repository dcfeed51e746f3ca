"""CPU oracle for the sketched-LUPP ID / CUR hot path.  TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
arm may import this module, and only as the checker (or the timed CPU
baseline).  The product path (paper_2310_09417_b200) never imports it.

This is a numpy/scipy restatement of the reference algorithm
(`/root/reference/pkg/src/randskel`, cited per function as file:line).  It is
*pinned* against the reference itself: tests/golden/make_golden.py imports
the reference from /root/reference (in the build container) and freezes its
outputs as fixtures; tests/test_oracle_golden.py checks this module against
them bit-for-bit on indices and to 1e-13 on values.

Algorithmic choices that matter for parity, restated:
  * LUPP pivot = first index of max |v| among the *current* positions of the
    active rows; full-row swaps; an exactly-zero pivot column stops the
    factorization (`dense.py:185-207`).  Panel width 64, blocked right-looking
    update with a unit-lower triangular solve + GEMM (`dense.py:210-233`).
  * Omega: numpy Philox4x64 keyed [seed, stream], C-order standard normals,
    ``/= sqrt(ell)`` for 'inv_sqrt_ell' (`sketching.py:55-72,191-204`).
  * Adaptive loop: block t uses child(t); estimate = ||S||_F of the Schur
    block; stop at e <= tau, or when rank + b > max_rank, or truncate on a
    zero pivot (`skeleton.py:391-460`).
"""

import numpy as np
import scipy.linalg

PANEL = 64            # dense.py:46
PINV_RCOND = 1e-12    # dense.py:49
COND_LIMIT = 1e14     # skeleton.py:72
_M64 = (1 << 64) - 1


class OracleRankDeficient(Exception):
    def __init__(self, step):
        super().__init__(step)
        self.step = step


# ---------------------------------------------------------------- streams --
def splitmix64(z):
    """`sketching.py:47-52`"""
    z = (z + 0x9E3779B97F4A7C15) & _M64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _M64
    return z ^ (z >> 31)


def child_stream(stream, i):
    """`sketching.py:71-72`: child(i) of stream id ``stream``."""
    return splitmix64((stream & _M64) ^ splitmix64(i & _M64))


def gaussian(seed, stream, n, ell, unit=False):
    """`sketching.py:191-204` with the key of `sketching.py:67-69`."""
    gen = np.random.Generator(np.random.Philox(key=[seed & _M64, stream & _M64]))
    om = gen.standard_normal((n, ell))
    if not unit:
        om /= np.sqrt(ell)
    return om


def srtt_dense(seed, stream, n, ell):
    """`sketching.py:134-157,207-216`: dense SRTT embedding (n x ell)."""
    import scipy.fft

    g = np.random.Generator(np.random.Philox(key=[seed & _M64, stream & _M64]))
    perm = g.permutation(n)
    signs = g.integers(0, 2, size=n) * 2.0 - 1.0
    cols = g.choice(n, size=ell, replace=False)
    eye = np.eye(n)
    c = scipy.fft.dct(eye[:, perm], type=2, axis=1, norm="ortho") * signs
    return np.sqrt(n / ell) * c[:, cols]


def srtt_operator(seed, stream, n, ell):
    """`sketching.py:207-216`: (perm, signs, cols, scale) of the SRTT embedding."""
    g = np.random.Generator(np.random.Philox(key=[seed & _M64, stream & _M64]))
    perm = g.permutation(n)
    signs = g.integers(0, 2, size=n) * 2.0 - 1.0
    cols = g.choice(n, size=ell, replace=False)
    return perm, signs, cols, np.sqrt(n / ell)


def srtt_apply(a, perm, signs, cols, scale):
    """`SrttSketch.apply` (`sketching.py:147-155`): scale * (DCT-II_ortho(a[:, perm]) * signs)[:, cols]."""
    import scipy.fft

    c = scipy.fft.dct(np.asarray(a, dtype=np.float64)[:, perm], type=2, axis=1, norm="ortho")
    c *= signs
    return scale * c[:, cols]


def sparse_sign_operator(seed, stream, n, ell, zeta):
    """`sketching.py:219-235`: (idx, signs, scale) of the sparse-sign embedding."""
    g = np.random.Generator(np.random.Philox(key=[seed & _M64, stream & _M64]))
    u = g.random((n, ell))
    idx = np.argsort(u, axis=1)[:, :zeta]
    signs = g.integers(0, 2, size=(n, zeta)) * 2.0 - 1.0
    return idx, signs, 1.0 / np.sqrt(zeta)


def sparse_sign_dense(seed, stream, n, ell, zeta):
    """`sketching.py:160-187,219-235`: dense sparse-sign embedding (n x ell)."""
    idx, signs, scale = sparse_sign_operator(seed, stream, n, ell, zeta)
    om = np.zeros((n, ell))
    np.put_along_axis(om, idx, signs / np.sqrt(zeta), axis=1)
    return om


def sparse_sign_apply(a, idx, signs, scale, ell):
    """`SparseSignSketch.apply` (`sketching.py:176-185`): ``(csr.T @ a.T).T`` in
    the order scipy's csc_matvecs evaluates it -- operator rows j ascending,
    ``y[:, c] += v * a[:, j]`` with ``v = signs * scale`` (a multiply, then an
    add), each y starting from zero."""
    a = np.asarray(a, dtype=np.float64)
    v = np.asarray(signs, dtype=np.float64) * scale
    y = np.zeros((a.shape[0], ell))
    for j in range(idx.shape[0]):
        for z in range(idx.shape[1]):
            c = idx[j, z]
            y[:, c] += v[j, z] * a[:, j]
    return y


# ------------------------------------------------------------------- LUPP --
def lupp_inplace(A, allow_partial):
    """Blocked right-looking LUPP of the F-ordered workspace A (m x n), in
    place.  Returns (perm, ncols).  `dense.py:185-233`."""
    m, n = A.shape
    perm = np.arange(m, dtype=np.intp)
    for c0 in range(0, n, PANEL):
        c1 = min(n, c0 + PANEL)
        for j in range(c0, c1):
            p = j + int(np.argmax(np.abs(A[j:, j])))
            if A[p, j] == 0.0:
                if allow_partial:
                    return perm, j
                raise OracleRankDeficient(j)
            if p != j:
                A[[j, p], :] = A[[p, j], :]
                perm[[j, p]] = perm[[p, j]]
            if j + 1 < m:
                A[j + 1:, j] /= A[j, j]
                if j + 1 < c1:
                    A[j + 1:, j + 1:c1] -= np.outer(A[j + 1:, j], A[j, j + 1:c1])
        if c1 < n:
            A[c0:c1, c1:] = scipy.linalg.solve_triangular(
                A[c0:c1, c0:c1], A[c0:c1, c1:], lower=True, unit_diagonal=True)
            A[c1:, c1:] -= A[c1:, c0:c1] @ A[c0:c1, c1:]
    return perm, n


def lupp(a, allow_partial=False):
    """(L, U, perm, ncols) with a[perm] = L U.  `dense.py:247-298`."""
    a = np.asarray(a, dtype=np.float64)
    m, n = a.shape
    if m < n:
        raise ValueError("lupp requires rows >= cols")
    if not np.isfinite(a).all():
        raise ValueError("non-finite entries")
    A = np.array(a, order="F", copy=True)
    perm, nc = lupp_inplace(A, allow_partial)
    L = np.tril(A[:, :nc], -1)
    L[np.arange(nc), np.arange(nc)] = 1.0
    U = np.triu(A[:nc, :nc])
    return L, U, perm, nc


def interp_from_lu(L, perm):
    """W with W[perm[:k]] = I, W[perm[k:]] = L2 L1^{-1}.  `skeleton.py:176-189`,
    right-side solve as `dense.py:553-560`."""
    k = L.shape[1]
    t = scipy.linalg.solve_triangular(L[:k], L[k:].T, lower=True, trans=1,
                                      unit_diagonal=True).T
    return scatter_interp(perm, k, t)


def scatter_interp(perm, k, t):
    w = np.zeros((perm.shape[0], k))
    w[perm[:k], np.arange(k)] = 1.0
    w[perm[k:]] = t
    return w


# ------------------------------------------------------- fixed-rank IDs --
def rand_lupp(a, k, seed, stream=0, unit=False):
    """`skeleton.py:207-234`: returns (row_idx, w)."""
    a = np.asarray(a, dtype=np.float64)
    om = gaussian(seed, stream, a.shape[1], k, unit)
    L, _, perm, _ = lupp(a @ om)
    return perm[:k].copy(), interp_from_lu(L, perm)


def column_id(a, k, seed, stream=0, unit=False):
    """`skeleton.py:574-589`: returns (col_idx, x)."""
    a = np.asarray(a, dtype=np.float64)
    gam = gaussian(seed, stream, a.shape[0], k, unit)
    L, _, perm, _ = lupp(a.T @ gam)
    return perm[:k].copy(), interp_from_lu(L, perm).T


# ----------------------------------------------------------- adaptive ID --
class LUState:
    """ysofar[perm] = [L1; L2] U1 (`skeleton.py:152-173`)."""

    def __init__(self, L1, L2, U1, perm, ysofar):
        self.L1, self.L2, self.U1, self.perm, self.ysofar = L1, L2, U1, perm, ysofar

    @property
    def rank(self):
        return self.U1.shape[0]


def block(a, seed, stream, t, b, zeta=None):
    """Sketch block t: a @ Omega_t, Omega_t ~ N(0, 1/b) from child(t)
    (`skeleton.py:286-295`); with ``zeta`` the sparse-sign block of the same
    stream (`_block_spec`: zeta capped at b), applied in scipy's SpMM order."""
    if zeta is not None:
        idx, sg, sc = sparse_sign_operator(seed, child_stream(stream, t), a.shape[1], b, min(zeta, b))
        return sparse_sign_apply(a, idx, sg, sc, b)
    return a @ gaussian(seed, child_stream(stream, t), a.shape[1], b)


def schur(state, y):
    """`skeleton.py:317-323`: (u2, S)."""
    k = state.rank
    py = y[state.perm]
    u2 = scipy.linalg.solve_triangular(state.L1, py[:k], lower=True, unit_diagonal=True)
    return u2, py[k:] - state.L2 @ u2


def extend(state, y, u2, L, U, sperm, nc):
    """`skeleton.py:326-351`."""
    if nc == 0:
        return state
    k = state.rank
    l2p = state.L2[sperm]
    L1 = np.block([[state.L1, np.zeros((k, nc))], [l2p[:nc], L[:nc]]])
    L2 = np.hstack([l2p[nc:], L[nc:]])
    U1 = np.block([[state.U1, u2[:, :nc]], [np.zeros((nc, k)), U]])
    perm = state.perm.copy()
    perm[k:] = perm[k:][sperm]
    return LUState(L1, L2, U1, perm, np.hstack([state.ysofar, y[:, :nc]]))


def adaptive_init(a, b, seed, stream=0, zeta=None):
    """`skeleton.py:298-314`."""
    y = block(a, seed, stream, 0, b, zeta)
    L, U, perm, _ = lupp(y)
    return LUState(L[:b].copy(), L[b:].copy(), U, perm, y)


RESIDUAL_STREAM = 1 << 40  # `skeleton.py:75`


def adaptive_step(state, a, b, seed, stream, t):
    """`skeleton.py:354-388` for block t: (e_schur, new state)."""
    y = block(a, seed, stream, t, b)
    u2, s = schur(state, y)
    e = float(np.linalg.norm(s))
    L, U, sperm, nc = lupp(s, allow_partial=True)
    return e, extend(state, y, u2, L, U, sperm, nc)


def draw_residual_sample(a, p, seed, stream=0):
    """`skeleton.py:527-539` (Gaussian): a @ Omega_r, unit-variance Omega_r from
    the stream's child(1 << 40)."""
    return a @ gaussian(seed, child_stream(stream, RESIDUAL_STREAM), a.shape[1], p, unit=True)


def residual_ur_estimates(state, a, p, seed, stream=0):
    """`skeleton.py:463-524` (Gaussian): norms of the trailing p x p factor of
    the dedicated sample, scaled by (4 log k / k) sqrt(m - k)."""
    m = a.shape[0]
    k = state.rank
    y_r = draw_residual_sample(a, p, seed, stream)
    _, s_r = schur(state, y_r)
    L, U, _, nc = lupp(s_r, allow_partial=True)
    norm_ur = float(np.linalg.norm(U)) if nc else 0.0
    max_ur = float(np.abs(U).max()) if nc else 0.0
    factor = (4.0 * np.log(k) / k) * np.sqrt(m - k)
    return dict(norm_ur=norm_ur, max_ur=max_ur, est_norm=factor * norm_ur, est_max=factor * max_ur)


def rand_lupp_adaptive(a, b, tau, seed, stream=0, max_rank=None, want_w=True, max_blocks=None, zeta=None):
    """`skeleton.py:391-460`: returns dict(rank, row_idx, w, trace, status).

    ``max_blocks`` (not in the reference) stops after that many sketch blocks
    -- the bounded CPU-baseline sample of bench.py.  ``zeta``: sparse-sign
    blocks with that many nonzeros per row instead of Gaussian ones."""
    a = np.asarray(a, dtype=np.float64)
    m, n = a.shape
    if max_rank is None:
        max_rank = max(b, min(m, n) - b)
    max_rank = min(max_rank, min(m, n))
    state = adaptive_init(a, b, seed, stream, zeta)
    trace, status, t = [], "not_converged", 1
    while max_blocks is None or t < max_blocks:
        y = block(a, seed, stream, t, b, zeta)
        u2, s = schur(state, y)
        e = float(np.linalg.norm(s))
        trace.append((state.rank, e))
        if e <= tau:
            status = "ok"
            break
        if state.rank + b > max_rank:
            break
        L, U, sperm, nc = lupp(s, allow_partial=True)
        state = extend(state, y, u2, L, U, sperm, nc)
        t += 1
        if nc < b:
            status = "rank_exhausted"
            break
    k = state.rank
    out = dict(rank=k, row_idx=state.perm[:k].copy(), trace=trace, status=status, state=state)
    if want_w:
        tb = scipy.linalg.solve_triangular(state.L1, state.L2.T, lower=True, trans=1,
                                           unit_diagonal=True).T
        out["w"] = scatter_interp(state.perm, k, tb)
    return out


# ------------------------------------------------------ two-sided / CUR --
def columns_from_rows(a, row_idx, k):
    """`skeleton.py:565-571`."""
    L, _, perm, _ = lupp(a[row_idx].T)
    return perm[:k].copy(), interp_from_lu(L, perm).T


def cond1(s):
    """1-norm condition estimate via getrf + gecon (`skeleton.py:592-603`)."""
    anorm = float(np.abs(s).sum(axis=0).max())
    if anorm == 0.0:
        return np.inf
    lu, _, info = scipy.linalg.lapack.dgetrf(s)
    if info > 0:
        return np.inf
    rc, _ = scipy.linalg.lapack.dgecon(lu, anorm, norm="1")
    return np.inf if rc == 0.0 else 1.0 / rc


def pinv_apply(a, b):
    """gelsd least squares, rcond 1e-12 (`dense.py:166-182`)."""
    b = np.asarray(b, dtype=np.float64)
    if b.ndim == 1:
        b = b[:, None]
    return scipy.linalg.lstsq(a, b, cond=PINV_RCOND, lapack_driver="gelsd")[0]


def two_sided_id(a, k, seed, stream=0):
    """`skeleton.py:606-625`."""
    a = np.asarray(a, dtype=np.float64)
    row_idx, w = rand_lupp(a, k, seed, stream)
    col_idx, x = columns_from_rows(a, row_idx, k)
    status = "ill_conditioned" if cond1(a[np.ix_(row_idx, col_idx)]) > COND_LIMIT else "ok"
    return dict(row_idx=row_idx, col_idx=col_idx, w=w, x=x, status=status)


def cur_from_rows(a, row_idx, k):
    """CUR assembly given row skeletons (`skeleton.py:637-647`)."""
    col_idx, _ = columns_from_rows(a, row_idx, k)
    c = a[:, col_idx]
    ar = pinv_apply(a[row_idx].T, a.T).T
    u_mid = pinv_apply(c, ar)
    status = "ill_conditioned" if cond1(a[np.ix_(row_idx, col_idx)]) > COND_LIMIT else "ok"
    return dict(row_idx=row_idx, col_idx=col_idx, u_mid=u_mid, status=status)


def cur_decompose(a, k, seed, stream=0):
    """`skeleton.py:628-647`."""
    a = np.asarray(a, dtype=np.float64)
    row_idx, _ = rand_lupp(a, k, seed, stream)
    return cur_from_rows(a, row_idx, k)


# --------------------------------------------------- evaluators / inputs --
def row_id_error(a, row_idx, w):
    """`skeleton.py:542-547`."""
    return float(np.linalg.norm(a - w @ a[row_idx]))


def stable_row_id_error(a, row_idx):
    """`skeleton.py:550-562`."""
    q, _ = np.linalg.qr(a[row_idx].T)
    at = a.T
    return float(np.linalg.norm(at - q @ (q.T @ at)))


def gen_fast_decay(m, n, beta, seed, stream=0):
    """Haar bases, singular values beta^((i-1)/(n-1)) (`zoo.py:36-75`)."""
    gen = np.random.Generator(np.random.Philox(key=[seed & _M64, stream & _M64]))

    def haar(r, c):
        q, rr = np.linalg.qr(gen.standard_normal((r, c)))
        s = np.sign(np.diagonal(rr))
        s[s == 0] = 1.0
        return q * s

    u = haar(m, n)
    v = haar(n, n)
    d = np.ones(1) if n == 1 else beta ** (np.arange(n) / (n - 1))
    return (u * d) @ v.T, d


def gen_kahan(n, zeta=0.99):
    """`zoo.py:78-88`."""
    phi = np.sqrt(1.0 - zeta * zeta)
    k = np.eye(n) - phi * np.triu(np.ones((n, n)), 1)
    return zeta ** np.arange(n)[:, None] * k


def gen_chan(n):
    """`zoo.py:91-104`."""
    a = np.eye(n) - np.tril(np.ones((n, n)), -1)
    a[:, -1] = 1.0
    return a


def fwht_rows(x, c, rowscale=None):
    """x <- rowscale * (c * H x), H acting on the row index, butterfly levels
    h = 1, 2, ..., n/2 (the device generator rs_fwht_rows, gen.cu)."""
    n = x.shape[0]
    h = 1
    while h < n:
        v = x.reshape(n // (2 * h), 2, h, x.shape[1])
        a = v[:, 0].copy()
        b = v[:, 1].copy()
        v[:, 0] = a + b
        v[:, 1] = a - b
        h *= 2
    x *= c
    if rowscale is not None:
        x *= rowscale[:, None]
    return x


def gen_fast_decay_hadamard(n, beta, seed, stream=0):
    """cfg5's input (paper_2310_09417_b200.zoo.gen_fast_decay_hadamard):
    A = (H S0 H S1) diag(d) (S3 H S2 H), H = Walsh-Hadamard / sqrt(n),
    signs from Generator(Philox(key=[seed, stream])).integers(0, 2, (4, n)).
    Same operations and rounding order as the device kernels."""
    gen = np.random.Generator(np.random.Philox(key=[seed & _M64, stream & _M64]))
    signs = gen.integers(0, 2, size=(4, n)).astype(np.float64) * 2.0 - 1.0
    d = np.ones(1) if n == 1 else beta ** (np.arange(n) / (n - 1))
    c = 1.0 / np.sqrt(n)
    x = fwht_rows(np.eye(n), c, signs[2])
    x = fwht_rows(x, c, signs[3] * d * signs[1])
    x = fwht_rows(x, c, signs[0])
    x = fwht_rows(x, c)
    return x, d


def cfg3_test_matrix(m, n, r=200, rel_noise=1e-6, seed=0):
    """cfg3's non-negative low-rank-plus-noise recipe at a checkable size,
    made bit-reproducible on any host: W, H have 8-bit dyadic entries in
    [0, 1) (so W @ H is exact whatever the BLAS), N is uniform [0, 1), the
    norms are exactly rounded (math.fsum) and the rest is elementwise IEEE.
    Returns the fp32 matrix (the reference upcasts it to fp64)."""
    import math

    g = np.random.default_rng(seed)
    w = g.integers(0, 256, size=(m, r)).astype(np.float64) / 256.0
    h = g.integers(0, 256, size=(r, n)).astype(np.float64) / 256.0
    low = w @ h
    noise = g.random((m, n))
    eta = rel_noise * math.sqrt(math.fsum((low * low).ravel())) / math.sqrt(math.fsum((noise * noise).ravel()))
    return (low + eta * noise).astype(np.float32)


def philox_uniform(seed, stream, shape):
    """numpy Generator(Philox(key=[seed, stream])).random(shape)."""
    return np.random.Generator(np.random.Philox(key=[seed & _M64, stream & _M64])).random(shape)


def exact_rank(m, n, r, seed):
    """`test_skeleton.py:12-14`."""
    g = np.random.default_rng(seed)
    return g.standard_normal((m, r)) @ g.standard_normal((r, n))
