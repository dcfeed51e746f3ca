"""Where and why the full-size cfg2 pivot sequences of the CUDA path and the oracle part.

Runs the CUDA path on the cfg2 matrix (bench.py's generator), finds the first pivot p0
where its row_idx differs from the oracle's, replays the oracle loop (oracle/randskel_oracle.py,
`skeleton.py:298-388`) up to the block that chooses p0, and at that block's Schur block S
(`skeleton.py:317-323`) reports:
  - the candidates' |S| at column c = p0 mod b after the oracle's own c elimination steps
    (`dense.py:185-207`): the top two values, their rows, and where the GPU's choice ranks;
  - the rounding level of S: S recomputed a second, independent way in fp64
    (py[k:] - Ysofar_p[k:] Ysofar_p[:k]^-1 py[:k], one LU solve of the k x k pivot block
    instead of the accumulated L-form), max |S - S_alt| / max |S|, and the pivot the
    second S picks at column c.
Test infrastructure (the oracle is the checker).

  python tools/cfg2_divergence.py --n 20000 --out gpurun_out/cfg2_divergence.json
"""
import argparse
import json
import os
import sys
import time

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
sys.path.insert(0, os.path.join(REPO, "oracle"))


def eliminate(s, cols):
    """The oracle's unblocked partial-pivoting steps 0..cols-1 on a copy of s;
    returns (S after the steps, row order)."""
    A = np.array(s, order="F", copy=True)
    order = np.arange(A.shape[0])
    for j in range(cols):
        p = j + int(np.argmax(np.abs(A[j:, j])))
        if p != j:
            A[[j, p], :] = A[[p, j], :]
            order[[j, p]] = order[[p, j]]
        A[j + 1:, j] /= A[j, j]
        A[j + 1:, j + 1:] -= np.outer(A[j + 1:, j], A[j, j + 1:])
    return A, order


def candidates(A, order, c, rows):
    v = np.abs(A[c:, c])
    ids = rows[order[c:]]
    top = np.argsort(-v, kind="stable")
    return v, ids, top


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=20000)
    ap.add_argument("--b", type=int, default=64)
    ap.add_argument("--tau", type=float, default=1e-8)
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--out", default=None)
    args = ap.parse_args()

    import torch
    from threadpoolctl import threadpool_limits

    import bench
    import paper_2310_09417_b200 as rs
    import randskel_oracle as orc

    dev = torch.device("cuda", 0)
    n, b = args.n, args.b
    a = bench.gen_fast_decay_device(n, 1e-16, args.seed, dev)
    res = rs.rand_lupp_adaptive(a.T, b, args.tau, rs.SketchSpec("gaussian", n, b), rs.RngStream(args.seed))
    g_idx = np.asarray(res.row_idx.cpu() if hasattr(res.row_idx, "cpu") else res.row_idx, dtype=np.int64)
    at = np.ascontiguousarray(a.cpu().numpy().T)
    del a
    torch.cuda.empty_cache()

    out = {"n": n, "b": b, "tau": args.tau}
    with threadpool_limits(limits=os.cpu_count() or 1):
        t0 = time.perf_counter()
        state = orc.adaptive_init(at, b, args.seed, 0)
        prev, B, t = None, None, 1
        if not np.array_equal(state.perm[:b], g_idx[:b]):
            B = 0
        while B is None and state.rank < len(g_idx):
            prev = state
            _, state = orc.adaptive_step(state, at, b, args.seed, 0, t)
            kk = min(state.rank, len(g_idx))
            if not np.array_equal(state.perm[:kk], g_idx[:kk]):
                B = t
            t += 1
        if B is None or B == 0:
            out["first_difference"] = None if B is None else "block 0"
            print(json.dumps(out))
            return
        state = prev
        k = state.rank
        # the oracle's new pivots come from the step's factorisation, not state.perm
        # of the previous state: recompute them below from S.
        y = orc.block(at, args.seed, 0, B, b)
        _, s = orc.schur(state, y)
        _, _, sperm, _ = orc.lupp(s, allow_partial=True)
        r_new = state.perm[k:][sperm][:b]
        c = int(np.nonzero(r_new != g_idx[k:k + b])[0][0])
        p0 = k + c
        out.update(first_difference=p0, block=B, column=c, gpu_row=int(g_idx[p0]), oracle_row=int(r_new[c]))
        yp = state.ysofar[state.perm]
        py = y[state.perm]
        s_alt = py[k:] - yp[k:] @ np.linalg.solve(yp[:k], py[:k])
        rows = state.perm[k:]
        out["replay_seconds"] = time.perf_counter() - t0

    out["k"] = int(k)
    out["S_max_abs"] = float(np.abs(s).max())
    out["S_rounding_level_rel"] = float(np.abs(s - s_alt).max() / np.abs(s).max())
    A1, o1 = eliminate(s, c)
    v, ids, top = candidates(A1, o1, c, rows)
    gpos = int(np.nonzero(ids == g_idx[p0])[0][0]) if (ids == g_idx[p0]).any() else -1
    rank_of_gpu = int(np.nonzero(top == gpos)[0][0]) if gpos >= 0 else -1
    out["oracle_S"] = {
        "top2_values": [float(v[top[0]]), float(v[top[1]])], "top2_rows": [int(ids[top[0]]), int(ids[top[1]])],
        "top2_rel_gap": float((v[top[0]] - v[top[1]]) / v[top[0]]),
        "gpu_choice_rank": rank_of_gpu, "gpu_choice_value": float(v[gpos]) if gpos >= 0 else None,
        "gpu_choice_rel_gap": float((v[top[0]] - v[gpos]) / v[top[0]]) if gpos >= 0 else None,
        "column_max_over_S_max": float(v[top[0]] / np.abs(s).max()),
    }
    A2, o2 = eliminate(s_alt, c)
    v2, ids2, top2 = candidates(A2, o2, c, rows)
    out["alt_S"] = {"top2_values": [float(v2[top2[0]]), float(v2[top2[1]])],
                    "top2_rows": [int(ids2[top2[0]]), int(ids2[top2[1]])],
                    "prefix_before_column_equal": bool(np.array_equal(o1[:c], o2[:c]))}
    line = json.dumps(out)
    print(line, flush=True)
    if args.out:
        with open(args.out, "w") as f:
            f.write(line + "\n")


if __name__ == "__main__":
    main()
