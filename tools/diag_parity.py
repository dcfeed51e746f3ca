"""Print parity diagnostics (prefix agreement, residuals) vs golden fixtures."""
import sys, os
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", "tests"))
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", "oracle"))
import numpy as np
import paper_2310_09417_b200 as rs
from conftest import golden
import randskel_oracle as orc

def prefix(a, b):
    n = min(len(a), len(b)); d = np.nonzero(a[:n] != b[:n])[0]
    return n if d.size == 0 else int(d[0])

for case in ["adapt_fd200", "adapt_fd150_s0", "adapt_fd150_s1", "adapt_fd150_s2", "adapt_notconv",
             "adapt_exhausted", "adapt_wide", "adapt_b25", "adapt_fullwidth", "adapt_single"]:
    g = golden(case); a = g["a"]; mr = int(g["max_rank"]); b = int(g["b"])
    res = rs.rand_lupp_adaptive(a, b, float(g["tau"]), rs.SketchSpec("gaussian", a.shape[1], b),
                                rs.RngStream(int(g["seed"])), max_rank=None if mr < 0 else mr)
    na = np.linalg.norm(a)
    e_ours = np.linalg.norm(a - res.w @ a[res.row_idx]) / na
    e_ref = np.linalg.norm(a - g["w"] @ a[g["row_idx"]]) / na
    tr = np.array([r.e_schur for r in res.trace])
    print(f"{case:18s} rank {res.rank}/{int(g['rank'])} prefix {prefix(res.row_idx, g['row_idx'])} "
          f"set {len(set(res.row_idx) & set(g['row_idx']))} W relerr "
          f"{np.linalg.norm(res.w - g['w']) / np.linalg.norm(g['w']):.2e} resid {e_ours:.3e} ref {e_ref:.3e} "
          f"dtrace {np.abs(tr - g['trace'][:, 1]).max() / na:.2e}")
a = golden("fast_decay_300")["a"]
for k in (40, 150):
    g = golden(f"rand_lupp_fd300_k{k}")
    r = rs.rand_lupp(a, k, rs.SketchSpec("gaussian", 300, 32), rs.RngStream(int(g["seed"])))
    na = np.linalg.norm(a)
    print(f"rand_lupp k{k} prefix {prefix(r.row_idx, g['row_idx'])} resid "
          f"{np.linalg.norm(a - r.w @ a[r.row_idx]) / na:.3e} ref {np.linalg.norm(a - g['w'] @ a[g['row_idx']]) / na:.3e}"
          f" W relerr {np.linalg.norm(r.w - g['w']) / np.linalg.norm(g['w']):.2e}")
g = golden("adapt_cfg2_n2000")
a, _ = orc.gen_fast_decay(2000, 2000, 1e-16, 0, orc.child_stream(0, 1 << 41))
res = rs.rand_lupp_adaptive(a.T, 64, 1e-8, rs.SketchSpec("gaussian", 2000, 64), rs.RngStream(0))
at = a.T
print("cfg2 n2000 rank", res.rank, "prefix", prefix(res.row_idx, g["row_idx"]), "resid",
      np.linalg.norm(at - res.w @ at[res.row_idx]) / np.linalg.norm(a),
      "w_sq", (res.w ** 2).sum(), float(g["w_sq"]), "w_sum", res.w.sum(), float(g["w_sum"]))
