"""Seeded random shapes through the public API vs the oracle: odd sizes,
k = 1, b = 1, b > 64, thin and wide matrices, numpy and torch inputs.
Random Gaussian matrices have well-separated pivots, so skeletons and pivot
order must be identical; W within the residual rule of test_gpu_parity."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

import randskel_oracle as orc  # noqa: E402

CASES = np.random.default_rng(2024).integers(0, 10**6, size=24)


def _shape(seed):
    g = np.random.default_rng(int(seed))
    m = int(g.integers(2, 400))
    n = int(g.integers(2, 400))
    return g, m, n


@pytest.mark.parametrize("seed", CASES[:12])
def test_fuzz_fixed_rank(seed):
    import paper_2310_09417_b200 as rs

    g, m, n = _shape(seed)
    a = g.standard_normal((m, n))
    k = int(g.integers(1, min(m, n) + 1))
    s = int(g.integers(0, 1000))
    r = rs.rand_lupp(a, k, rs.SketchSpec("gaussian", n, k), rs.RngStream(s))
    ridx, w = orc.rand_lupp(a, k, s)
    assert np.array_equal(r.row_idx, ridx)
    assert np.allclose(r.w, w, rtol=1e-9, atol=1e-9 * max(1.0, np.abs(w).max()))
    c = rs.column_id(torch.as_tensor(a), k, rs.SketchSpec("gaussian", m, k), rs.RngStream(s))
    cidx, x = orc.column_id(a, k, s)
    assert np.array_equal(c.col_idx.numpy(), cidx)


@pytest.mark.parametrize("seed", CASES[12:])
def test_fuzz_adaptive(seed):
    import paper_2310_09417_b200 as rs

    g, m, n = _shape(seed)
    r0 = int(g.integers(1, min(m, n) + 1))
    a = g.standard_normal((m, r0)) @ g.standard_normal((r0, n)) + 1e-3 * g.standard_normal((m, n))
    b = int(g.choice([1, 3, 16, 64, 100]))
    b = min(b, min(m, n))
    tau = float(10 ** g.uniform(-2, 1)) * np.sqrt(m * n) * 1e-3
    s = int(g.integers(0, 1000))
    res = rs.rand_lupp_adaptive(a, b, tau, rs.SketchSpec("gaussian", n, b), rs.RngStream(s))
    ref = orc.rand_lupp_adaptive(a, b, tau, s)
    assert res.status == ref["status"]
    assert res.rank == ref["rank"]
    assert np.array_equal(res.row_idx, ref["row_idx"])
    tr = np.array([t.e_schur for t in res.trace])
    tr_ref = np.array([t[1] for t in ref["trace"]])
    assert np.allclose(tr, tr_ref, rtol=1e-9, atol=1e-12 * np.linalg.norm(a))
    na = np.linalg.norm(a)
    if res.rank:
        e = np.linalg.norm(a - res.w @ a[res.row_idx]) / na
        e_ref = np.linalg.norm(a - ref["w"] @ a[ref["row_idx"]]) / na
        assert e <= 1.5 * e_ref + 1e-13
