"""Full-size proof of the summation-order contract: the adaptive column ID
gives the same bits -- every e_schur, every pivot, the rank -- whether A is a device tensor, a
pageable numpy array, a pinned numpy array (host inputs go through the chunked pre-sketch), or
column-sharded (the N > 1 code path) at world size 1.

  python tools/determinism_full.py --cfg 2        # 20000^2 Haar fast decay (bench.py's matrix)
  python tools/determinism_full.py --cfg 5        # 65536^2 randomized-Hadamard fast decay

Writes one JSON line per variant plus a summary line.
"""
import argparse
import json
import os
import sys
import time

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cfg", type=int, default=2)
    ap.add_argument("--n", type=int, default=None)
    ap.add_argument("--host", action="store_true", help="also the pageable / pinned numpy inputs")
    args = ap.parse_args()
    import torch
    import torch.distributed as dist

    import paper_2310_09417_b200 as rs
    from paper_2310_09417_b200.sharded import rand_lupp_adaptive_sharded

    if args.cfg == 2:
        from bench import gen_fast_decay_device

        n = args.n or 20000
        a = gen_fast_decay_device(n, 1e-16, 0, torch.device("cuda", 0))
    else:
        n = args.n or 65536
        a, _ = rs.gen_fast_decay_hadamard(n, 1e-16, rs.RngStream(0).child(1 << 41))
    torch.cuda.synchronize()
    spec = rs.SketchSpec("gaussian", n, 64)
    runs = {}

    def record(name, fn):
        torch.cuda.synchronize()
        t0 = time.time()
        res = fn()
        torch.cuda.synchronize()
        dt = time.time() - t0
        idx = res.row_idx.cpu().numpy() if isinstance(res.row_idx, torch.Tensor) else np.asarray(res.row_idx)
        tr = [(t.k, t.e_schur) for t in res.trace]
        runs[name] = (res.rank, idx, tr, res.status)
        print(json.dumps({"variant": name, "n": n, "rank": res.rank, "blocks": len(tr) + 1, "status": res.status,
                          "seconds": round(dt, 3)}), flush=True)
        del res

    record("device", lambda: rs.rand_lupp_adaptive(a.T, 64, 1e-8, spec, rs.RngStream(0)))
    dist.init_process_group("gloo", store=dist.HashStore(), rank=0, world_size=1)
    try:
        record("sharded_world1", lambda: rand_lupp_adaptive_sharded(a.T, 64, 1e-8, spec, rs.RngStream(0)))
    finally:
        dist.destroy_process_group()
    if args.host:
        h = a.cpu().numpy()  # C-ordered A; the column ID runs on its transposed view
        del a
        torch.cuda.empty_cache()
        record("numpy_pageable", lambda: rs.rand_lupp_adaptive(h.T, 64, 1e-8, spec, rs.RngStream(0)))
        hp = torch.from_numpy(h).pin_memory().numpy()
        del h
        record("numpy_pinned", lambda: rs.rand_lupp_adaptive(hp.T, 64, 1e-8, spec, rs.RngStream(0)))
    ref = runs["device"]
    summary = {}
    for name, (k, idx, tr, st) in runs.items():
        summary[name] = {"rank_equal": k == ref[0], "pivots_equal": bool(np.array_equal(idx, ref[1])),
                         "trace_bits_equal": tr == ref[2], "status_equal": st == ref[3]}
    print(json.dumps({"cfg": args.cfg, "n": n, "rank": ref[0], "bitwise_vs_device": summary,
                      "all_equal": all(all(v.values()) for v in summary.values())}), flush=True)


if __name__ == "__main__":
    main()
