import sys, numpy as np, torch
sys.path.insert(0, ".")
import bench, paper_2310_09417_b200 as rs
from paper_2310_09417_b200.sharded import rand_lupp_adaptive_sharded
for n in (6000, 20000):
    a = bench.gen_fast_decay_device(n, 1e-16, 0, torch.device("cuda", 0))
    spec = rs.SketchSpec("gaussian", n, 64)
    r1 = rs.rand_lupp_adaptive(a.T, 64, 1e-8, spec, rs.RngStream(0))
    r2 = rand_lupp_adaptive_sharded(a.T, 64, 1e-8, spec, rs.RngStream(0))
    i1, i2 = r1.row_idx.cpu().numpy(), r2.row_idx.cpu().numpy()
    m = min(len(i1), len(i2)); d = np.nonzero(i1[:m] != i2[:m])[0]
    t1 = np.array([r.e_schur for r in r1.trace]); t2 = np.array([r.e_schur for r in r2.trace])
    k = min(len(t1), len(t2)); first = int(np.nonzero(t1[:k] != t2[:k])[0][0]) if (t1[:k] != t2[:k]).any() else None
    print(n, "ranks", r1.rank, r2.rank, "prefix", m if d.size == 0 else int(d[0]), "first trace entry not bitwise", first,
          "max rel dtrace", float(np.max(np.abs(t1[:k] - t2[:k]) / t1[:k])))
