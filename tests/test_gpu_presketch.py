"""Host inputs >= 64 MB: the first blocks are sketched while A is copied in
(`skeleton._presketch`); results must match the plain path (same skeletons,
rank, status; traces and W to rounding) for C- and F-ordered inputs, and the
plain path must match the oracle."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

import randskel_oracle as orc  # noqa: E402


@pytest.mark.parametrize("order", ["C", "F"])
def test_presketch_matches_plain_path(order, monkeypatch):
    import paper_2310_09417_b200 as rs

    a, _ = orc.gen_fast_decay(3200, 3000, 1e-14, 5, 1)
    a = np.asarray(a, order=order)
    assert a.nbytes >= 64 << 20
    tau = 1e-9 * np.linalg.norm(a)
    spec = rs.SketchSpec("gaussian", a.shape[1], 64)
    out = {}
    for mode in ("1", "0"):
        monkeypatch.setenv("RSKEL_PRESKETCH", mode)
        out[mode] = rs.rand_lupp_adaptive(a, 64, tau, spec, rs.RngStream(9))
    r1, r0 = out["1"], out["0"]
    assert r1.rank == r0.rank and r1.status == r0.status
    assert np.array_equal(r1.row_idx, r0.row_idx)
    t1 = np.array([t.e_schur for t in r1.trace])
    t0 = np.array([t.e_schur for t in r0.trace])
    assert np.allclose(t1, t0, rtol=1e-9, atol=1e-12 * np.linalg.norm(a))
    na = np.linalg.norm(a)
    e1 = np.linalg.norm(a - r1.w @ a[r1.row_idx]) / na
    e0 = np.linalg.norm(a - r0.w @ a[r0.row_idx]) / na
    assert e1 <= 1.5 * e0 + 1e-13


@pytest.mark.parametrize("order", ["C", "F"])
def test_streamed_fixed_rank_matches_plain_path(order, monkeypatch):
    import paper_2310_09417_b200 as rs

    g = np.random.default_rng(3)
    a = np.asarray(g.standard_normal((3000, 2900)), order=order)
    out = {}
    for mode in ("1", "0"):
        monkeypatch.setenv("RSKEL_PRESKETCH", mode)
        out[mode] = (rs.column_id(a, 200, rs.SketchSpec("gaussian", 3000, 200), rs.RngStream(4)),
                     rs.rand_lupp(a, 150, rs.SketchSpec("gaussian", 2900, 150), rs.RngStream(5)))
    (c1, r1), (c0, r0) = out["1"], out["0"]
    assert np.array_equal(c1.col_idx, c0.col_idx)
    assert np.allclose(c1.x, c0.x, rtol=1e-9, atol=1e-9)
    assert np.array_equal(r1.row_idx, r0.row_idx)
    assert np.allclose(r1.w, r0.w, rtol=1e-9, atol=1e-9)
    cidx, _ = orc.column_id(a, 200, 4)
    assert np.array_equal(c1.col_idx, cidx)
