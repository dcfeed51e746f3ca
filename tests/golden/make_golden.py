"""Freeze golden vectors from the REAL reference (build container only).

Imports `randskel` from /root/reference/pkg/src (read-only, never copied) and
records its outputs on seeded inputs as compressed .npz fixtures under
tests/golden/.  The fixtures pin the oracle (tests/test_oracle_golden.py) and
are the parity targets of the GPU tests (tests/test_gpu_parity.py).  The GPU
box has no /root/reference; it only reads these files.

Run:  python tests/golden/make_golden.py
"""

import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
OUT = os.path.dirname(os.path.abspath(__file__))


def main():
    sys.path.insert(0, REF)
    import randskel as rs
    from randskel.skeleton import _column_skeletons_from_rows

    cases = {}

    def put(name, **arrays):
        cases[name] = arrays

    def spec(n, ell=None):
        return rs.SketchSpec("gaussian", n=n, ell=ell or min(n, 32))

    def exact(m, n, r, seed):
        g = np.random.default_rng(seed)
        return g.standard_normal((m, r)) @ g.standard_normal((r, n))

    # ---- LUPP known answers ------------------------------------------------
    f = rs.lupp(np.array([[1, 5], [1, 5], [3, 0], [1, 1]], dtype=float))
    put("lupp_tiebreak", perm=f.perm, L=f.L, U=f.U)
    f = rs.lupp([[1, 2], [3, 4]])
    put("lupp_hand", perm=f.perm, L=f.L, U=f.U)
    for n in (5, 10, 20, 30):
        f = rs.lupp(rs.gen_chan(n))
        put(f"lupp_chan{n}", perm=f.perm, L=f.L, U=f.U)
    for seed, (m, k) in enumerate([(30, 17), (40, 25), (300, 100), (1000, 200), (700, 130)]):
        # input regenerated in the tests from default_rng(seed).standard_normal((m, k))
        a = np.random.default_rng(seed).standard_normal((m, k))
        f = rs.lupp(a)
        if m <= 40:
            put(f"lupp_rand{seed}", m=m, k=k, perm=f.perm, L=f.L, U=f.U)
        else:
            put(f"lupp_rand{seed}", m=m, k=k, perm=f.perm, L_sum=f.L.sum(), U_sum=f.U.sum(),
                L_head=f.L[:64].copy(), U_head=f.U[:16].copy())

    # ---- fixed-rank row / column ID ----------------------------------------
    a = exact(120, 80, 30, 0)
    r = rs.rand_lupp(a, 30, spec(80), rs.RngStream(1))
    put("rand_lupp_exact", a=a, k=30, seed=1, ell_spec=32, row_idx=r.row_idx, w=r.w)

    a, sig = rs.gen_fast_decay(300, 300, 1e-16, rs.RngStream(99))
    put("fast_decay_300", a=a, sigma=sig)
    for k, seed in ((40, 3), (150, 2)):
        r = rs.rand_lupp(a, k, spec(300), rs.RngStream(seed))
        put(f"rand_lupp_fd300_k{k}", k=k, seed=seed, row_idx=r.row_idx, w=r.w,
            resid=np.linalg.norm(a - r.w @ a[r.row_idx]) / np.linalg.norm(a))
        c = rs.column_id(a, k, spec(300), rs.RngStream(seed))
        put(f"column_id_fd300_k{k}", k=k, seed=seed, col_idx=c.col_idx, x=c.x,
            resid=np.linalg.norm(a - a[:, c.col_idx] @ c.x) / np.linalg.norm(a))

    a = exact(80, 60, 20, 47)
    c = rs.column_id(a, 20, spec(60), rs.RngStream(48))
    put("column_id_exact", a=a, k=20, seed=48, col_idx=c.col_idx, x=c.x)

    # column ID at 1000 x 1000, k = 256 (cfg1 shape scaled down)
    a, sig = rs.gen_fast_decay(1000, 1000, 1e-16, rs.RngStream(5))
    c = rs.column_id(a, 256, rs.SketchSpec("gaussian", 1000, 256), rs.RngStream(0))
    put("column_id_fd1000_k256", gen_seed=5, col_idx=c.col_idx, x_sum=c.x.sum(),
        x_sq=(c.x ** 2).sum(), x_head=c.x[:, :16].copy(), a_sum=a.sum(),
        resid=np.linalg.norm(a - a[:, c.col_idx] @ c.x) / np.linalg.norm(a))

    # ---- adaptive --------------------------------------------------------
    def adaptive(name, mat, b, tau, seed, max_rank=None, keep_w=True, **extra):
        res = rs.rand_lupp_adaptive(mat, b, tau, spec(mat.shape[1], b), rs.RngStream(seed),
                                    max_rank=max_rank)
        tr = np.array([[rec.k, rec.e_schur] for rec in res.trace])
        resid = np.linalg.norm(mat - res.w @ mat[res.row_idx]) / np.linalg.norm(mat)
        d = dict(b=b, tau=tau, seed=seed, max_rank=-1 if max_rank is None else max_rank,
                 rank=res.rank, row_idx=res.row_idx, trace=tr, status=res.status, resid=resid,
                 **extra)
        if keep_w:
            d["w"] = res.w
        else:
            d["w_sum"] = res.w.sum()
            d["w_sq"] = (res.w ** 2).sum()
            d["w_head"] = res.w[:16].copy()
        put(name, **d)

    a, _ = rs.gen_fast_decay(200, 200, 1e-16, rs.RngStream(24))
    adaptive("adapt_fd200", a, 20, 1e-4 * np.linalg.norm(a), 25, a=a)
    a, _ = rs.gen_fast_decay(150, 150, 1e-16, rs.RngStream(26))
    for s in range(3):
        adaptive(f"adapt_fd150_s{s}", a, 15, 1e-13 * np.linalg.norm(a), s, a=a)
    a, _ = rs.gen_fast_decay(80, 80, 1e-4, rs.RngStream(27))
    adaptive("adapt_notconv", a, 10, 1e-30, 28, max_rank=40, a=a)
    g = np.random.default_rng(29)
    a = np.zeros((50, 40))
    a[:12] = g.standard_normal((12, 40))
    adaptive("adapt_exhausted", a, 8, 1e-30, 30, a=a)
    a_tall, _ = rs.gen_fast_decay(240, 90, 1e-12, rs.RngStream(60))
    a = a_tall.T.copy()
    adaptive("adapt_wide", a, 15, 1e-6 * np.linalg.norm(a), 61, a=a)
    a, _ = rs.gen_fast_decay(100, 100, 1e-16, rs.RngStream(33))
    adaptive("adapt_b25", a, 25, 1e-5 * np.linalg.norm(a), 34, a=a)
    a, _ = rs.gen_fast_decay(30, 20, 1e-8, rs.RngStream(12))
    adaptive("adapt_fullwidth", a, 20, 1e-14, 13, a=a)
    a, _ = rs.gen_fast_decay(100, 80, 1e-12, rs.RngStream(22))
    adaptive("adapt_single", a, 16, 2 * np.linalg.norm(a), 23, a=a)

    # criterion-4 matrix (1000^2, b=50): detection at rank 650 / 350
    a, _ = rs.gen_fast_decay(1000, 1000, 1e-16, rs.RngStream(500))
    na = np.linalg.norm(a)
    for tau_rel in (1e-8, 1e-4):
        adaptive(f"adapt_crit4_{tau_rel:g}", a, 50, tau_rel * na, 0, keep_w=False, gen_seed=500)
    # b = 64, absolute tau = 1e-8 as cfg2, on a 2000 x 2000 fast-decay matrix (column ID: a.T)
    a, _ = rs.gen_fast_decay(2000, 2000, 1e-16, rs.RngStream(0).child(1 << 41))
    adaptive("adapt_cfg2_n2000", np.ascontiguousarray(a.T), 64, 1e-8, 0, keep_w=False,
             gen_seed=0, a_sum=a.sum())

    # max_rank below the block size: the first block is still absorbed whole
    a, _ = rs.gen_fast_decay(120, 100, 1e-12, rs.RngStream(90))
    adaptive("adapt_maxrank0", a, 16, 1e-30, 91, max_rank=0, a=a)
    adaptive("adapt_maxrank15", a, 16, 1e-30, 92, max_rank=15, a=a)

    # ---- two-sided / CUR ---------------------------------------------------
    a = exact(80, 60, 20, 49)
    r = rs.two_sided_id(a, 20, spec(60), rs.RngStream(50))
    put("two_sided_exact", a=a, k=20, seed=50, row_idx=r.row_idx, col_idx=r.col_idx, w=r.w,
        x=r.x, status=r.status)
    a = exact(75, 55, 18, 53)
    cur = rs.cur_decompose(a, 18, spec(55), rs.RngStream(54))
    put("cur_exact", a=a, k=18, seed=54, row_idx=cur.row_idx, col_idx=cur.col_idx,
        u_mid=cur.u_mid, status=cur.status)
    a, _ = rs.gen_fast_decay(300, 300, 1e-16, rs.RngStream(99))
    cur = rs.cur_decompose(a, 100, spec(300), rs.RngStream(55))
    put("cur_fd300", k=100, seed=55, row_idx=cur.row_idx, col_idx=cur.col_idx,
        u_mid=cur.u_mid, status=cur.status)
    r = rs.two_sided_id(np.diag([1.0] * 5 + [1e-16] * 5), 8, spec(10), rs.RngStream(57))
    put("two_sided_illcond", row_idx=r.row_idx, col_idx=r.col_idx, status=r.status)
    # cond_1 flag: a matrix whose dgecon estimate (7.4e13) and exact 1-norm condition
    # number (1.03e14) straddle the 1e14 limit (skeleton.py:592-603)
    from randskel.skeleton import _condition_estimate_1norm
    g = np.random.default_rng(0)
    for _ in range(4000):
        n = int(g.integers(20, 60))
        q1, _ = np.linalg.qr(g.standard_normal((n, n)))
        q2, _ = np.linalg.qr(g.standard_normal((n, n)))
        c = 10 ** g.uniform(12.5, 14.5)
        smat = (q1 * np.logspace(0, -np.log10(c), n)) @ q2.T
        est = _condition_estimate_1norm(smat)
        kappa = np.abs(smat).sum(0).max() * np.abs(np.linalg.inv(smat)).sum(0).max()
        if est < 1e14 < kappa:
            put("cond1_straddle", s=smat, est=est, exact=kappa)
            break
    # adaptive-CUR composition (cfg3 recipe at 1024 x 512)
    g = np.random.default_rng(0)
    wmat = g.random((1024, 100))
    hmat = g.random((100, 512))
    low = wmat @ hmat
    noise = g.random((1024, 512))
    eta = 1e-6 * np.linalg.norm(low) / np.linalg.norm(noise)
    a = (low + eta * noise).astype(np.float32).astype(np.float64)
    tau = 1e-5 * np.linalg.norm(a)
    res = rs.rand_lupp_adaptive(a, 64, tau, spec(512, 64), rs.RngStream(0))
    col_idx, _ = _column_skeletons_from_rows(a, res.row_idx, res.rank)
    put("adaptive_cur_nonneg", tau=tau, rank=res.rank,
        row_idx=res.row_idx, col_idx=col_idx, status=res.status,
        trace=np.array([[rec.k, rec.e_schur] for rec in res.trace]))

    # ---- residual-U_r certificates and error evaluators --
    a, _ = rs.gen_fast_decay(400, 300, 1e-12, rs.RngStream(70))
    st = rs.adaptive_init(a, 16, spec(300, 16), rs.RngStream(71))
    for _ in range(3):
        _, st = rs.adaptive_step(st, a, spec(300, 16))
    for p in (4, 15):
        y_r = rs.draw_residual_sample(a, p, spec(300, 16), rs.RngStream(72))
        est = rs.residual_ur_estimates(st, a, p, spec(300, 16), rs.RngStream(72))
        put(f"resid_ur_p{p}", gen_seed=70, b=16, steps=3, seed=71, rseed=72, p=p, rank=st.rank,
            perm=st.perm, y_r_sum=y_r.sum(), norm_ur=est.norm_ur, max_ur=est.max_ur,
            est_norm=est.est_norm, est_max=est.est_max)
    r = rs.rand_lupp(a, 48, spec(300, 48), rs.RngStream(73))
    put("row_id_errors", gen_seed=70, k=48, seed=73, row_idx=r.row_idx,
        err=rs.row_id_error(a, r), stable_err=rs.stable_row_id_error(a, r))

    # ---- structured embeddings: SRTT and sparse sign ----
    a = np.random.default_rng(80).standard_normal((90, 70))
    for kind, kw in (("srtt", {}), ("sparsesign", {"zeta": 4})):
        sp = rs.SketchSpec(kind, n=70, ell=16, **kw)
        op = rs.make_sketch(sp, rs.RngStream(81))
        put(f"sketch_{kind}", dense=op.to_dense(), y=rs.apply_sketch(a, op),
            yt=rs.apply_sketch(a, rs.make_sketch(rs.SketchSpec(kind, n=90, ell=16, **kw), rs.RngStream(82)),
                               side="transposed_right"))
        r = rs.rand_lupp(a, 16, rs.SketchSpec(kind, n=70, ell=16, **kw), rs.RngStream(83))
        put(f"rand_lupp_{kind}", row_idx=r.row_idx, w=r.w)
        b_exact = exact(120, 90, 25, 84)
        res = rs.rand_lupp_adaptive(b_exact, 8, 1e-9, rs.SketchSpec(kind, n=90, ell=8, **kw), rs.RngStream(85))
        put(f"adapt_{kind}", rank=res.rank, row_idx=res.row_idx, status=res.status,
            trace=np.array([[rec.k, rec.e_schur] for rec in res.trace]))

    path = os.path.join(OUT, "reference_golden.npz")
    _save(cases, path)
    configs()


def _save(cases, path):
    flat = {}
    for name, arrays in cases.items():
        for key, val in arrays.items():
            flat[f"{name}/{key}"] = np.asarray(val)
    np.savez_compressed(path, **flat)
    print(f"wrote {len(cases)} cases, {os.path.getsize(path) / 1e6:.2f} MB -> {path}")


def configs():
    """BASELINE.json configs at checkable sizes, from the reference itself
    (tests/test_gpu_configs.py): cfg1 at its full size, cfg4's Kahan matrix at
    4096 with k = 512 (+ the CPQR comparator), cfg3's recipe at 4096 x 2048,
    cfg5's device generator at 8192 (the oracle's numpy restatement of the
    randomized-Hadamard construction, bit-identical to the device one)."""
    sys.path.insert(0, REF)
    sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(OUT)), "oracle"))
    import randskel as rs
    import randskel_oracle as orc
    from randskel.skeleton import _column_skeletons_from_rows

    cases = {}

    def put(name, **arrays):
        cases[name] = arrays

    # cfg1: column ID of the 4096^2 fast-decay matrix, k = 256 (BASELINE configs[0])
    a, _ = rs.gen_fast_decay(4096, 4096, 1e-16, rs.RngStream(0).child(1 << 41))
    c = rs.column_id(a, 256, rs.SketchSpec("gaussian", 4096, 256), rs.RngStream(0))
    put("cfg1_full", col_idx=c.col_idx, x_sum=c.x.sum(), x_sq=(c.x ** 2).sum(), x_head=c.x[:, :16].copy(),
        a_sum=a.sum(), resid=np.linalg.norm(a - a[:, c.col_idx] @ c.x) / np.linalg.norm(a))
    del a, c

    # cfg4: Kahan (zeta 0.99) at 4096, k = 512: LUPP vs CPQR skeletons (pivot robustness)
    a = rs.gen_kahan(4096, 0.99)
    sp = rs.SketchSpec("gaussian", 4096, 512)
    c = rs.column_id(a, 512, sp, rs.RngStream(0))
    r = rs.rand_lupp(a, 512, sp, rs.RngStream(0))
    q = rs.rand_cpqr(a, 512, sp, rs.RngStream(0))
    put("cfg4_kahan4096", col_idx=c.col_idx, x_sum=c.x.sum(), x_sq=(c.x ** 2).sum(), row_idx=r.row_idx,
        w_sum=r.w.sum(), w_sq=(r.w ** 2).sum(), stable_err=rs.stable_row_id_error(a, r),
        cpqr_row_idx=q.row_idx, cpqr_stable_err=rs.stable_row_id_error(a, q),
        col_resid=np.linalg.norm(a - a[:, c.col_idx] @ c.x) / np.linalg.norm(a))
    del a, c, r, q

    # cfg3 recipe at 4096 x 2048 (fp32 input, the reference upcasts): adaptive CUR
    a32 = orc.cfg3_test_matrix(4096, 2048)
    a = a32.astype(np.float64)
    tau = 1e-5 * np.linalg.norm(a)
    res = rs.rand_lupp_adaptive(a, 64, tau, rs.SketchSpec("gaussian", 2048, 64), rs.RngStream(0))
    k = res.rank
    col_idx, _ = _column_skeletons_from_rows(a, res.row_idx, k)
    cmat = a[:, col_idx]
    rows = a[res.row_idx]
    u_mid = rs.pinv_apply(cmat, rs.pinv_apply(rows.T, a.T).T)   # skeleton.py:639-646 with k = rank
    put("cfg3_cur4096", a32_sum=a.sum(), a32_head=a32[:4, :64].copy(), tau=tau, rank=k, row_idx=res.row_idx, col_idx=col_idx, u_mid=u_mid,
        status=res.status, trace=np.array([[rec.k, rec.e_schur] for rec in res.trace]),
        resid=np.linalg.norm(a - cmat @ u_mid @ rows) / np.linalg.norm(a))
    del a, a32, cmat, rows

    # cfg5 recipe at 8192: randomized-Hadamard fast decay, adaptive column ID b = 64, tau = 1e-8
    n = 8192
    gen = rs.RngStream(0).child(1 << 41)
    a, _ = orc.gen_fast_decay_hadamard(n, 1e-16, gen.seed, gen.stream)
    res = rs.rand_lupp_adaptive(np.ascontiguousarray(a.T), 64, 1e-8, rs.SketchSpec("gaussian", n, 64),
                                rs.RngStream(0))
    put("cfg5_hadamard8192", a_sum=a.sum(), a_sq=(a ** 2).sum(), a_head=a[:4, :64].copy(), rank=res.rank,
        row_idx=res.row_idx, status=res.status, trace=np.array([[rec.k, rec.e_schur] for rec in res.trace]))
    path = os.path.join(OUT, "config_golden.npz")
    _save(cases, path)


if __name__ == "__main__":
    if sys.argv[1:] == ["--configs"]:
        configs()
    else:
        main()
