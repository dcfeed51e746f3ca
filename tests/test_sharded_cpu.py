"""Column-sharded adaptive loop at world_size 2 and 3 over gloo on CPU.

The per-rank arithmetic is the CPU test double (tests/shard_cpu_ops.py); what
is under test is the sharded host logic of `paper_2310_09417_b200.sharded`:
ownership maps, the three exact all-reduces per block, the replicated panel
and stop rule.  Every rank must return the oracle's single-process result
(`oracle/randskel_oracle.py:rand_lupp_adaptive`, the restatement of
`skeleton.py:391-460`): same skeletons in the same pivot order, same rank,
status and trace; the rank's rows of W match the oracle's W.
"""

import os
import socket
import sys

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(HERE)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _matrix(kind, m, n, seed):
    sys.path.insert(0, os.path.join(REPO, "oracle"))
    import randskel_oracle as orc

    if kind == "decay":
        a, _ = orc.gen_fast_decay(m, n, 1e-12, seed, 77)
        return a
    # 12 nonzero rows spread over the ranks: the Schur block dies exactly
    # (`test_skeleton.py:208-218`) -> rank_exhausted at 12
    g = np.random.default_rng(seed)
    a = np.zeros((m, n))
    a[np.arange(0, m, 5)[:12]] = g.standard_normal((12, n))
    return a


def _worker(rank, world, port, case, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    sys.path[:0] = [REPO, HERE]
    import torch.distributed as dist

    import paper_2310_09417_b200 as rs
    from paper_2310_09417_b200.sharded import rand_lupp_adaptive_sharded
    from shard_cpu_ops import CpuShardOps

    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        kind, m, n, b, tau, seed, counts, max_rank = case[:8]
        sk = case[8] if len(case) > 8 else "gaussian"
        a = _matrix(kind, m, n, seed)
        lo = sum(counts[:rank])
        hi = lo + counts[rank]
        ops = CpuShardOps(a[lo:hi], seed)
        spec = rs.SketchSpec(sk, n, b, **({"zeta": 4} if sk == "sparsesign" else {}))
        res = rand_lupp_adaptive_sharded(a[lo:hi], b, tau, spec, rs.RngStream(seed), max_rank=max_rank, ops=ops)
        q.put((rank, res.rank, np.asarray(res.row_idx), res.status,
               [(r.k, r.e_schur) for r in res.trace], np.asarray(res.w)))
    except Exception as e:  # surface worker failures in the parent
        q.put((rank, "error", repr(e)))
        raise
    finally:
        dist.destroy_process_group()


CASES = [
    # kind, m, n, b, tau, seed, rows per rank, max_rank
    ("decay", 240, 160, 8, 1e-6, 3, [100, 140], None),        # converges: status ok
    ("decay", 240, 160, 8, 1e-6, 3, [60, 120, 60], None),     # 3 ranks, uneven
    ("zero_rows", 60, 40, 8, 1e-30, 5, [25, 35], None),       # rank_exhausted at 12
    ("decay", 200, 150, 16, 1e-14, 1, [10, 190], 96),          # not_converged at max_rank
    # b > 64: each block factored as 64-column panels (the paper's b = 128)
    ("decay", 400, 300, 96, 1e-6, 3, [150, 250], None),       # panels 64 + 32, converges
    ("decay", 420, 380, 128, 1e-14, 1, [420], 256),           # one rank, not_converged at max_rank
    ("decay", 420, 380, 128, 1e-14, 1, [100, 200, 120], 256),  # three ranks, same case
]


def _run_world(case):
    import torch.multiprocessing as mp

    world = len(case[6])
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, case, q)) for r in range(world)]
    for p in procs:
        p.start()
    outs = {}
    try:
        for _ in range(world):
            item = q.get(timeout=240)
            assert item[1] != "error", item
            outs[item[0]] = item
    finally:
        for p in procs:
            p.join(timeout=60)
            if p.is_alive():
                p.kill()
    return outs


@pytest.mark.parametrize("sk", ["sparsesign", "srtt"])
def test_sharded_structured_sketch_world_invariant(sk):
    """SRTT / sparse-sign blocks in the sharded loop: every rank applies the same
    per-block operator to its rows, so 1 and 3 ranks give the same skeleton,
    trace bits and W."""
    base = ("decay", 300, 200, 16, 1e-8, 6)
    one = _run_world(base + ([300], None, sk))
    three = _run_world(base + ([90, 110, 100], None, sk))
    _, k1, r1, s1, t1, w1 = one[0]
    assert k1 > 16 and len(t1) >= 2
    for r in range(3):
        _, k, ri, st, tr, _ = three[r]
        assert (k, st, tr) == (k1, s1, t1)
        assert np.array_equal(ri, r1)
    assert np.array_equal(np.vstack([three[r][5] for r in range(3)]), w1)


@pytest.mark.parametrize("case", CASES, ids=["ok-2", "ok-3-uneven", "exhausted-2", "maxrank-2", "wide96-2",
                                             "wide128-1", "wide128-3"])
def test_sharded_matches_oracle(case):
    import torch.multiprocessing as mp

    sys.path.insert(0, os.path.join(REPO, "oracle"))
    import randskel_oracle as orc

    kind, m, n, b, tau, seed, counts, max_rank = case
    world = len(counts)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, case, q)) for r in range(world)]
    for p in procs:
        p.start()
    outs = {}
    try:
        for _ in range(world):
            item = q.get(timeout=240)
            assert item[1] != "error", item
            outs[item[0]] = item
    finally:
        for p in procs:
            p.join(timeout=60)
            if p.is_alive():
                p.kill()
    a = _matrix(kind, m, n, seed)
    ref = orc.rand_lupp_adaptive(a, b, tau, seed, max_rank=max_rank)
    k = ref["rank"]
    w_parts = []
    for r in range(world):
        _, kk, row_idx, status, trace, w = outs[r]
        assert kk == k
        assert status == ref["status"]
        assert np.array_equal(row_idx, ref["row_idx"])
        assert [t[0] for t in trace] == [t[0] for t in ref["trace"]]
        np.testing.assert_allclose([t[1] for t in trace], [t[1] for t in ref["trace"]], rtol=1e-7, atol=1e-12)
        w_parts.append(w)
    w = np.vstack(w_parts)
    assert w.shape == ref["w"].shape
    assert np.array_equal(w[ref["row_idx"]], np.eye(k))
    # W is ill-conditioned in its trailing columns near the noise floor: compare
    # the interpolation residual ||a - W a[row_idx]|| (as tests/test_gpu_parity.py)
    na = np.linalg.norm(a)
    res = np.linalg.norm(a - w @ a[ref["row_idx"]]) / na
    res_ref = np.linalg.norm(a - ref["w"] @ a[ref["row_idx"]]) / na
    assert res <= 1.5 * res_ref + 1e-13, (res, res_ref)
    np.testing.assert_allclose(w, ref["w"], rtol=0, atol=1e-6 * max(1.0, np.abs(ref["w"]).max()))
