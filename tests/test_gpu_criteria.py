"""Reference acceptance properties on the device path: the Schur-block estimator is
unbiased (reference `tests/test_skeleton.py:131-147`, criterion 3), and the adaptive loop's
skeletons are the one-shot LUPP prefix of the concatenated blocks (`test_skeleton.py:221-232`,
criterion 2)."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def rs():
    import paper_2310_09417_b200 as rs

    return rs


@pytest.mark.parametrize("kind", ["gaussian", "srtt", "sparsesign"])
def test_estimator_unbiased_within_standard_errors(rs, kind):
    a, _ = rs.gen_fast_decay(100, 100, 1e-16, rs.RngStream(20))
    spec = rs.SketchSpec(kind, n=100, ell=20)
    state = rs.adaptive_init(a, 20, spec, rs.RngStream(21))
    w = rs.interpolation_matrix(state)
    truth = np.linalg.norm(a - w @ a[state.perm[:20]]) ** 2
    draws = np.empty(300)
    for i in range(draws.size):
        e, _ = rs.adaptive_step(state, a, spec, rs.RngStream(5000).child(i))
        draws[i] = e ** 2
    se = draws.std(ddof=1) / np.sqrt(draws.size)
    assert abs(draws.mean() - truth) <= 5 * se


def test_adaptive_equals_one_shot_prefix(rs):
    from paper_2310_09417_b200 import _device
    from paper_2310_09417_b200.lu_state import _draw_block

    a, _ = rs.gen_fast_decay(120, 100, 1e-16, rs.RngStream(31))
    spec = rs.SketchSpec("gaussian", n=100, ell=100)
    res = rs.rand_lupp_adaptive(a, b=10, tau=1e-6 * np.linalg.norm(a), spec=spec, rng=rs.RngStream(32))
    A = _device.as_matrix(a)
    blocks = [_draw_block(A, spec, rs.RngStream(32).child(t), 10).cpu().numpy() for t in range(res.rank // 10)]
    one = rs.lupp(np.hstack(blocks))
    assert np.array_equal(res.row_idx, one.perm[: res.rank])


def _gaussian_spec(rs, n, ell=None):
    return rs.SketchSpec("gaussian", n=n, ell=ell or min(n, 32))  # the reference helper (test_skeleton.py:8-9)


def _exact_rank_matrix(m, n, r, seed):
    g = np.random.default_rng(seed)
    return g.standard_normal((m, r)) @ g.standard_normal((r, n))


def test_adaptive_init_shapes_and_determinism(rs):
    """Reference `test_skeleton.py:77-86`."""
    a, _ = rs.gen_fast_decay(60, 40, 1e-10, rs.RngStream(10))
    spec = _gaussian_spec(rs, 40)
    s1 = rs.adaptive_init(a, 8, spec, rs.RngStream(11))
    s2 = rs.adaptive_init(a, 8, spec, rs.RngStream(11))
    assert s1.L1.shape == (8, 8)
    assert np.array_equal(np.diagonal(s1.L1), np.ones(8))
    assert np.abs(np.tril(s1.L1, -1)).max() <= 1 + 1e-14
    assert np.array_equal(s1.perm, s2.perm)
    assert np.array_equal(s1.ysofar, s2.ysofar)


def test_adaptive_init_full_width_boundary(rs):
    """Reference `test_skeleton.py:89-96`: the first block spans the factorable width."""
    a, _ = rs.gen_fast_decay(30, 20, 1e-8, rs.RngStream(12))
    res = rs.rand_lupp_adaptive(a, b=20, tau=1e-14, spec=_gaussian_spec(rs, 20), rng=rs.RngStream(13))
    assert res.rank == 20
    assert len(res.trace) == 1


def test_adaptive_step_exact_rank_small_estimate(rs):
    """Reference `test_skeleton.py:99-105`."""
    a = _exact_rank_matrix(80, 60, 10, 14)
    spec = _gaussian_spec(rs, 60)
    state = rs.adaptive_init(a, 12, spec, rs.RngStream(15))
    e, state2 = rs.adaptive_step(state, a, spec)
    assert e <= 1e-10 * np.linalg.norm(a)
    assert state2.rank == 24


def test_adaptive_rank_detection_scaled(rs):
    """Reference `test_skeleton.py:176-183`."""
    a, _ = rs.gen_fast_decay(200, 200, 1e-16, rs.RngStream(24))
    na = np.linalg.norm(a)
    res = rs.rand_lupp_adaptive(a, b=20, tau=1e-4 * na, spec=_gaussian_spec(rs, 200), rng=rs.RngStream(25))
    assert res.status == rs.STATUS_OK
    assert 40 <= res.rank <= 80
    assert rs.row_id_error(a, res) <= 3 * 1e-4 * na


def test_adaptive_trace_monotone_on_decaying_spectra(rs):
    """Reference `test_skeleton.py:186-195`: >= 95 % of seeded runs have a monotone trace."""
    a, _ = rs.gen_fast_decay(150, 150, 1e-16, rs.RngStream(26))
    spec = _gaussian_spec(rs, 150)
    monotone = 0
    for seed in range(20):
        res = rs.rand_lupp_adaptive(a, b=15, tau=1e-13 * np.linalg.norm(a), spec=spec, rng=rs.RngStream(seed))
        vals = [rec.e_schur for rec in res.trace]
        monotone += all(b <= a_ for a_, b in zip(vals, vals[1:]))
    assert monotone >= 19


# --------------------------------------------------- reference test_dense.py on the device ---
def test_lupp_matches_lapack_pivots(rs):
    """Reference `test_dense.py:154-167`: LAPACK getrf picks the same first-maximum pivots."""
    import scipy.linalg

    for seed in range(8):
        a = np.random.default_rng(seed).standard_normal((40, 25))
        f = rs.lupp(a)
        lu, piv = scipy.linalg.lu_factor(a)
        perm = np.arange(40)
        for i, p in enumerate(piv):
            perm[[i, p]] = perm[[p, i]]
        assert np.array_equal(f.perm, perm)
        assert np.abs(f.L - (np.tril(lu[:, :25], -1) + np.eye(40, 25))).max() <= 1e-13
        assert np.abs(f.U - np.triu(lu[:25, :25])).max() <= 1e-13


def test_lupp_bitwise_deterministic(rs):
    """Reference `test_dense.py:170-176`."""
    a = np.random.default_rng(77).standard_normal((60, 30))
    f1, f2 = rs.lupp(a), rs.lupp(a)
    assert np.array_equal(f1.L, f2.L) and np.array_equal(f1.U, f2.U) and np.array_equal(f1.perm, f2.perm)


@pytest.mark.parametrize("m,k,seed", [(20, 10, 0), (100, 60, 1), (300, 100, 2), (2, 1, 3), (24, 24, 4)])
def test_lupp_reconstruction(rs, m, k, seed):
    """Reference `test_dense.py:186-205` (shapes and the property test's bounds)."""
    eps = np.finfo(float).eps
    a = np.random.default_rng(seed).standard_normal((m, k))
    f = rs.lupp(a)
    assert np.linalg.norm(a[f.perm] - f.L @ f.U) <= 1e-12 * np.linalg.norm(a) * m
    assert np.abs(np.tril(f.L, -1)).max(initial=0.0) <= 1 + 16 * eps


@pytest.mark.parametrize("n", [2, 5, 10, 20, 30])
def test_chan_growth_factor_tight(rs, n):
    """Reference `test_dense.py:446-451`: growth exactly 2^(n-1), ties keep the first row."""
    eps = np.finfo(float).eps
    a = rs.gen_chan(n)
    f = rs.lupp(a)
    growth = np.abs(f.U).max() / np.abs(a).max()
    assert abs(growth - 2.0 ** (n - 1)) <= 4 * eps * 2.0 ** (n - 1)
    assert np.array_equal(f.perm, np.arange(n))


def test_pinv_apply_reference_cases(rs):
    """Reference `test_dense.py:422-433`: the null direction is truncated; normal equations hold."""
    x = rs.pinv_apply(np.diag([2.0, 0.0]), [[2.0], [2.0]])
    assert np.abs(np.asarray(x) - np.array([[1.0], [0.0]])).max() <= 1e-12
    g = np.random.default_rng(17)
    a = g.standard_normal((10, 4))
    b = g.standard_normal((10, 2))
    x = np.asarray(rs.pinv_apply(a, b))
    assert np.abs(a.T @ (a @ x - b)).max() <= 1e-12


# --------------------------------------------- reference test_acceptance.py on the device ---
def test_criterion_01_lu_factorization_correctness(rs):
    """Reference `test_acceptance.py:36-58`, the LU half (CPQR is the reference's
    comparator, not on the hot path): 100 factorizations, scaled residual <= 1e-12."""
    eps = np.finfo(float).eps
    shapes = [(20, 10), (100, 60), (300, 100)]
    worst_lu, worst_l = 0.0, 0.0
    for i in range(100):
        m, k = shapes[i % 3]
        a = np.random.default_rng(i).standard_normal((m, k))
        f = rs.lupp(a)
        worst_lu = max(worst_lu, np.linalg.norm(a[f.perm] - f.L @ f.U) / (np.linalg.norm(a) * m))
        worst_l = max(worst_l, np.abs(np.tril(f.L, -1)).max())
    assert worst_lu <= 1e-12 and worst_l <= 1 + 16 * eps


def test_criterion_06_growth_factor_bound(rs):
    """Reference `test_acceptance.py:185-214`: svd tail / ||U_r||_F estimate <=
    (4 log k / k) sqrt(m - k) at every rank of 20 seeded adaptive runs."""
    a, sigma = rs.gen_fast_decay(500, 500, 1e-16, rs.RngStream(888))
    m, p = 500, 10
    violations, points = 0, set()
    for seed in range(20):
        rng = rs.RngStream(seed)
        spec = rs.SketchSpec("gaussian", n=500, ell=45)
        state = rs.adaptive_init(a, 45, spec, rng)
        y_r = rs.draw_residual_sample(a, p, spec, rng)
        while True:
            k = state.rank
            est = rs.residual_ur_estimates(state, a, p, spec, rng, sample_r=y_r)
            tail = float(np.sqrt(np.sum(np.asarray(sigma)[k:] ** 2)))  # svd_tail_norm (dense.py:499)
            points.add(k)
            if tail / est.norm_ur > (4 * np.log(k) / k) * np.sqrt(m - k):
                violations += 1
            if k + 45 > 450:
                break
            _, state = rs.adaptive_step(state, a, spec)
    assert violations == 0 and len(points) == 10


def test_criterion_08_sketch_isometry(rs):
    """Reference `test_acceptance.py:235-256`: 10^4 draws per kind."""
    x = np.random.default_rng(31337).standard_normal((8, 64))
    nx2 = np.linalg.norm(x) ** 2
    for kind in ("gaussian", "srtt", "sparsesign"):
        spec = rs.SketchSpec(kind, n=64, ell=16, zeta=8)
        base = rs.RngStream(hash(kind) & 0xFFFF)
        total = 0.0
        for i in range(10_000):
            op = rs.make_sketch(spec, base.child(i))
            total += np.linalg.norm(np.asarray(rs.apply_sketch(x, op))) ** 2
        assert 0.95 <= total / 10_000 / nx2 <= 1.05, kind


def test_criterion_10_exact_rank_recovery(rs):
    """Reference `test_acceptance.py:279-313` for the five hot-path methods (CPQR aside)."""
    for r, seed in ((10, 1), (40, 2)):
        g = np.random.default_rng(seed)
        a = g.standard_normal((150, r)) @ g.standard_normal((r, 120))
        na = np.linalg.norm(a)
        spec = rs.SketchSpec("gaussian", n=120, ell=r)
        rng = rs.RngStream(seed)
        rl = rs.rand_lupp(a, r, spec, rng.child(1))
        errs = [np.linalg.norm(a - rl.w @ a[rl.row_idx])]
        ra = rs.rand_lupp_adaptive(a, b=r // 2, tau=1e-9 * na, spec=spec, rng=rng.child(3))
        assert ra.rank == r
        errs.append(np.linalg.norm(a - ra.w @ a[ra.row_idx]))
        rc = rs.column_id(a, r, spec, rng.child(4))
        errs.append(np.linalg.norm(a - a[:, rc.col_idx] @ rc.x))
        rt = rs.two_sided_id(a, r, spec, rng.child(5))
        errs.append(np.linalg.norm(a - rt.w @ a[np.ix_(rt.row_idx, rt.col_idx)] @ rt.x))
        cur = rs.cur_decompose(a, r, spec, rng.child(6))
        errs.append(np.linalg.norm(a - a[:, cur.col_idx] @ cur.u_mid @ a[cur.row_idx]))
        assert max(errs) <= 1e-8 * na, (r, errs)
