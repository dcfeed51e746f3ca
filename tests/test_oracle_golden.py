"""Pin the CPU oracle (oracle/randskel_oracle.py) to the reference's own outputs.

The golden fixtures were produced by importing the real reference package
(tests/golden/make_golden.py); the oracle is a from-scratch restatement of
its algorithm.  Indices and statuses must match exactly; values to 1e-12
relative (different BLAS call shapes round differently); the adaptive
estimates to 1e-13 * ||A||_F absolute.
"""

import numpy as np
import pytest

import randskel_oracle as orc
from conftest import golden


def relerr(x, y):
    return np.linalg.norm(np.asarray(x) - np.asarray(y)) / max(np.linalg.norm(y), 1e-300)


@pytest.mark.parametrize("case,mat", [
    ("lupp_tiebreak", [[1, 5], [1, 5], [3, 0], [1, 1]]),
    ("lupp_hand", [[1, 2], [3, 4]]),
])
def test_lupp_known_answers(case, mat):
    g = golden(case)
    L, U, perm, nc = orc.lupp(np.array(mat, dtype=float))
    assert np.array_equal(perm, g["perm"])
    assert np.array_equal(L, g["L"]) and np.array_equal(U, g["U"])


def test_tiebreak_is_current_position():
    # first maximum in the *current* position, not original index.
    _, _, perm, _ = orc.lupp(np.array([[1, 5], [1, 5], [3, 0], [1, 1]], dtype=float))
    assert perm.tolist() == [2, 1, 0, 3]


@pytest.mark.parametrize("n", [5, 10, 20, 30])
def test_lupp_chan_growth(n):
    g = golden(f"lupp_chan{n}")
    a = orc.gen_chan(n)
    L, U, perm, _ = orc.lupp(a)
    assert np.array_equal(perm, g["perm"]) and np.array_equal(perm, np.arange(n))
    assert np.array_equal(U, g["U"])
    assert np.abs(U).max() / np.abs(a).max() == 2.0 ** (n - 1)


@pytest.mark.parametrize("seed", range(5))
def test_lupp_random(seed):
    g = golden(f"lupp_rand{seed}")
    m, k = int(g["m"]), int(g["k"])
    a = np.random.default_rng(seed).standard_normal((m, k))
    L, U, perm, _ = orc.lupp(a)
    assert np.array_equal(perm, g["perm"])
    if "L" in g:
        assert np.abs(L - g["L"]).max() <= 1e-13 and np.abs(U - g["U"]).max() <= 1e-13
    else:
        assert abs(L.sum() - float(g["L_sum"])) <= 1e-9 * max(1.0, abs(float(g["L_sum"])))
        assert np.abs(L[:64] - g["L_head"]).max() <= 1e-12
        assert np.abs(U[:16] - g["U_head"]).max() <= 1e-11 * np.abs(g["U_head"]).max()


def test_lupp_zero_pivot_step():
    col0 = np.array([4.0, 2.0, 8.0, 1.0])
    col1 = np.array([1.0, 2.0, 4.0, 8.0])
    with pytest.raises(orc.OracleRankDeficient) as exc:
        orc.lupp(np.column_stack([col0, col1, col0]))
    assert exc.value.step == 2


def test_gaussian_streams_match_reference_rng():
    # child-stream derivation + Philox draw: the exact-rank row ID is a pure
    # function of them; compare its skeleton and W.
    g = golden("rand_lupp_exact")
    idx, w = orc.rand_lupp(g["a"], 30, seed=1)
    assert np.array_equal(idx, g["row_idx"])
    assert relerr(w, g["w"]) < 1e-12


@pytest.mark.parametrize("k", [40, 150])
def test_fixed_rank_ids(k):
    a = golden("fast_decay_300")["a"]
    g = golden(f"rand_lupp_fd300_k{k}")
    idx, w = orc.rand_lupp(a, k, seed=int(g["seed"]))
    assert np.array_equal(idx, g["row_idx"])
    assert relerr(w, g["w"]) < 1e-8
    g = golden(f"column_id_fd300_k{k}")
    cidx, x = orc.column_id(a, k, seed=int(g["seed"]))
    assert np.array_equal(cidx, g["col_idx"])
    assert relerr(x, g["x"]) < 1e-8


def test_fast_decay_generator_matches_reference():
    a, sig = orc.gen_fast_decay(300, 300, 1e-16, 99)
    g = golden("fast_decay_300")
    assert np.array_equal(sig, g["sigma"])
    assert np.abs(a - g["a"]).max() <= 1e-14


ADAPTIVE = ["adapt_fd200", "adapt_fd150_s0", "adapt_fd150_s1", "adapt_fd150_s2", "adapt_notconv",
            "adapt_exhausted", "adapt_wide", "adapt_b25", "adapt_fullwidth", "adapt_single", "adapt_maxrank0",
            "adapt_maxrank15"]


@pytest.mark.parametrize("case", ADAPTIVE)
def test_adaptive(case):
    g = golden(case)
    a = g["a"]
    mr = int(g["max_rank"])
    out = orc.rand_lupp_adaptive(a, int(g["b"]), float(g["tau"]), int(g["seed"]),
                                 max_rank=None if mr < 0 else mr)
    assert out["status"] == str(g["status"])
    assert out["rank"] == int(g["rank"])
    assert np.array_equal(out["row_idx"], g["row_idx"])
    tr = np.array(out["trace"])
    assert np.array_equal(tr[:, 0], g["trace"][:, 0])
    assert np.abs(tr[:, 1] - g["trace"][:, 1]).max() <= 1e-13 * np.linalg.norm(a)
    resid = np.linalg.norm(a - out["w"] @ a[out["row_idx"]]) / np.linalg.norm(a)
    assert abs(resid - float(g["resid"])) <= 1e-3 * float(g["resid"]) + 1e-14


@pytest.mark.parametrize("tau_rel", ["1e-08", "0.0001"])
def test_adaptive_criterion4(tau_rel):
    """The reference's documented 'known red' ranks (650 / 350) are reproduced."""
    g = golden(f"adapt_crit4_{tau_rel}")
    a, _ = orc.gen_fast_decay(1000, 1000, 1e-16, int(g["gen_seed"]))
    out = orc.rand_lupp_adaptive(a, 50, float(g["tau"]), 0, want_w=False)
    assert out["rank"] == int(g["rank"]) == (650 if tau_rel == "1e-08" else 350)
    assert np.array_equal(out["row_idx"], g["row_idx"])


def test_two_sided_and_cur():
    g = golden("two_sided_exact")
    out = orc.two_sided_id(g["a"], 20, seed=50)
    assert np.array_equal(out["row_idx"], g["row_idx"])
    assert np.array_equal(out["col_idx"], g["col_idx"])
    assert out["status"] == str(g["status"])
    g = golden("cur_exact")
    out = orc.cur_decompose(g["a"], 18, seed=54)
    assert np.array_equal(out["row_idx"], g["row_idx"]) and np.array_equal(out["col_idx"], g["col_idx"])
    assert relerr(out["u_mid"], g["u_mid"]) < 1e-8
    g = golden("two_sided_illcond")
    out = orc.two_sided_id(np.diag([1.0] * 5 + [1e-16] * 5), 8, seed=57)
    assert out["status"] == str(g["status"]) == "ill_conditioned"


def test_adaptive_cur_composition():
    g = golden("adaptive_cur_nonneg")
    rng = np.random.default_rng(0)
    wmat, hmat = rng.random((1024, 100)), rng.random((100, 512))
    low = wmat @ hmat
    noise = rng.random((1024, 512))
    a = (low + 1e-6 * np.linalg.norm(low) / np.linalg.norm(noise) * noise).astype(np.float32).astype(np.float64)
    out = orc.rand_lupp_adaptive(a, 64, float(g["tau"]), 0, want_w=False)
    assert out["rank"] == int(g["rank"]) and out["status"] == str(g["status"])
    assert np.array_equal(out["row_idx"], g["row_idx"])
    cidx, _ = orc.columns_from_rows(a, out["row_idx"], out["rank"])
    assert np.array_equal(cidx, g["col_idx"])


def test_adaptive_cfg2_recipe_n2000():
    """cfg2 recipe (column ID via A.T, b=64, absolute tau=1e-8) at n=2000."""
    g = golden("adapt_cfg2_n2000")
    a, _ = orc.gen_fast_decay(2000, 2000, 1e-16, 0, orc.child_stream(0, 1 << 41))
    assert abs(a.sum() - float(g["a_sum"])) < 1e-9
    out = orc.rand_lupp_adaptive(a.T, 64, 1e-8, 0)
    assert out["rank"] == int(g["rank"]) == 1344 and out["status"] == "ok"
    assert np.array_equal(out["row_idx"], g["row_idx"])
    resid = np.linalg.norm(a.T - out["w"] @ a.T[out["row_idx"]]) / np.linalg.norm(a)
    assert abs(resid - float(g["resid"])) <= 1e-2 * float(g["resid"])


@pytest.mark.parametrize("p", [4, 15])
def test_oracle_residual_ur_estimates(p):
    """Residual-U_r certificates (`skeleton.py:463-539`) vs the reference."""
    g = golden(f"resid_ur_p{p}")
    a, _ = orc.gen_fast_decay(400, 300, 1e-12, int(g["gen_seed"]))
    st = orc.adaptive_init(a, int(g["b"]), int(g["seed"]))
    for t in range(1, int(g["steps"]) + 1):
        _, st = orc.adaptive_step(st, a, int(g["b"]), int(g["seed"]), 0, t)
    assert st.rank == int(g["rank"])
    assert np.array_equal(st.perm, g["perm"])
    y_r = orc.draw_residual_sample(a, p, int(g["rseed"]))
    assert abs(y_r.sum() - float(g["y_r_sum"])) <= 1e-9 * np.abs(y_r).sum()
    est = orc.residual_ur_estimates(st, a, p, int(g["rseed"]))
    for key in ("norm_ur", "max_ur", "est_norm", "est_max"):
        assert abs(est[key] - float(g[key])) <= 1e-9 * abs(float(g[key])) + 1e-300, key


def test_oracle_row_id_errors():
    g = golden("row_id_errors")
    a, _ = orc.gen_fast_decay(400, 300, 1e-12, int(g["gen_seed"]))
    r = orc.rand_lupp(a, int(g["k"]), int(g["seed"]))
    assert np.array_equal(r[0], g["row_idx"])
    e = orc.row_id_error(a, r[0], r[1])
    s = orc.stable_row_id_error(a, r[0])
    assert abs(e - float(g["err"])) <= 1e-8 * float(g["err"])
    assert abs(s - float(g["stable_err"])) <= 1e-8 * float(g["stable_err"])


@pytest.mark.parametrize("kind", ["srtt", "sparsesign"])
def test_oracle_structured_embeddings(kind):
    """SRTT / sparse-sign operators (`sketching.py:134-235`) vs the reference."""
    g = golden(f"sketch_{kind}")
    om = orc.srtt_dense(81, 0, 70, 16) if kind == "srtt" else orc.sparse_sign_dense(81, 0, 70, 16, 4)
    np.testing.assert_allclose(om, g["dense"], rtol=0, atol=1e-14)
    a = np.random.default_rng(80).standard_normal((90, 70))
    np.testing.assert_allclose(a @ om, g["y"], rtol=0, atol=1e-12)


def test_oracle_sparse_sign_spmm_order_is_the_references():
    """The oracle's SpMM restatement (csc_matvecs order: rows ascending, multiply
    then add) reproduces the reference's `SparseSignSketch.apply` bit for bit,
    on both application sides (golden `y`, `yt`)."""
    g = golden("sketch_sparsesign")
    a = np.random.default_rng(80).standard_normal((90, 70))
    idx, signs, scale = orc.sparse_sign_operator(81, 0, 70, 16, 4)
    assert np.array_equal(orc.sparse_sign_apply(a, idx, signs, scale, 16), g["y"])
    idx, signs, scale = orc.sparse_sign_operator(82, 0, 90, 16, 4)
    assert np.array_equal(orc.sparse_sign_apply(a.T, idx, signs, scale, 16), g["yt"])


def test_oracle_srtt_apply_is_the_references():
    """The oracle's SRTT application (per-row DCT) reproduces the reference's golden y / yt."""
    g = golden("sketch_srtt")
    a = np.random.default_rng(80).standard_normal((90, 70))
    assert np.array_equal(orc.srtt_apply(a, *orc.srtt_operator(81, 0, 70, 16)), g["y"])
    assert np.array_equal(orc.srtt_apply(a.T, *orc.srtt_operator(82, 0, 90, 16)), g["yt"])


def test_oracle_sparse_sign_adaptive_matches_reference():
    """The oracle's adaptive loop with sparse-sign blocks reproduces the reference's
    golden case (rank, status, pivots, trace)."""
    ga = golden("adapt_sparsesign")
    gg = np.random.default_rng(84)
    b_exact = gg.standard_normal((120, 25)) @ gg.standard_normal((25, 90))
    r = orc.rand_lupp_adaptive(b_exact, 8, 1e-9, 85, zeta=4)
    assert r["rank"] == int(ga["rank"]) and r["status"] == str(ga["status"])
    assert np.array_equal(r["row_idx"], ga["row_idx"])
    np.testing.assert_allclose(np.array(r["trace"]), ga["trace"], rtol=1e-12, atol=1e-12 * ga["trace"][0, 1])


def test_cond1_estimate_straddles_limit():
    """The oracle's cond_1 is dgecon's estimate (skeleton.py:592-603), not the exact
    1-norm condition number: on this matrix they fall on opposite sides of 1e14."""
    g = golden("cond1_straddle")
    est = orc.cond1(g["s"])
    assert abs(est - float(g["est"])) <= 1e-10 * float(g["est"])
    assert est < 1e14 < float(g["exact"])
