"""Column-sharded adaptive loop on the device (librskel.so kernels).

world_size 1, 2 and 3 must reproduce the single-GPU `rand_lupp_adaptive` bit
for bit (the GEMM summation order depends on K alone, the exchanges are
exact).  world_size > 1 runs processes on the one visible GPU with the gloo
backend (host-staged collectives: the ranks' kernels never wait on each
other); skeletons, pivot order, rank, status and every trace bit must equal
the single-GPU run's, and its W rows must match.
"""

import os
import socket
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(HERE)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _matrix(m, n, seed):
    sys.path.insert(0, os.path.join(REPO, "oracle"))
    import randskel_oracle as orc

    a, _ = orc.gen_fast_decay(m, n, 1e-14, seed, 9)
    return a


def _single(a, b, tau, seed):
    import paper_2310_09417_b200 as rs

    spec = rs.SketchSpec("gaussian", a.shape[1], b)
    return rs.rand_lupp_adaptive(a, b, tau, spec, rs.RngStream(seed))


@pytest.mark.parametrize("b", [64, 128, 96])
def test_sharded_world1_bitwise_equals_single(b):
    """b = 64 (one panel per block) and b > 64 (64-column panels per block, the
    paper's b = 128)."""
    import torch.distributed as dist

    import paper_2310_09417_b200 as rs
    from paper_2310_09417_b200.sharded import rand_lupp_adaptive_sharded

    a = _matrix(700, 500, 2)
    tau = 1e-9 * np.linalg.norm(a)
    ref = _single(a, b, tau, 4)
    store = dist.HashStore()
    dist.init_process_group("gloo", store=store, rank=0, world_size=1)
    try:
        spec = rs.SketchSpec("gaussian", 500, b)
        got = rand_lupp_adaptive_sharded(a, b, tau, spec, rs.RngStream(4))
    finally:
        dist.destroy_process_group()
    assert got.rank == ref.rank and got.status == ref.status
    assert np.array_equal(got.row_idx, ref.row_idx)
    assert [(r.k, r.e_schur) for r in got.trace] == [(r.k, r.e_schur) for r in ref.trace]
    assert np.array_equal(got.w, ref.w)


@pytest.mark.parametrize("sk", ["sparsesign", "srtt"])
def test_sharded_structured_world1_bitwise_equals_single(sk):
    """SRTT / sparse-sign blocks: the sharded loop applies the reference's per-block
    operator to its rows (sparse sign through the SpMM) exactly as the single-GPU loop."""
    import torch.distributed as dist

    import paper_2310_09417_b200 as rs
    from paper_2310_09417_b200.sharded import rand_lupp_adaptive_sharded

    a = _matrix(600, 450, 3)
    tau = 1e-9 * np.linalg.norm(a)
    kw = {"zeta": 6} if sk == "sparsesign" else {}
    ref = rs.rand_lupp_adaptive(a, 48, tau, rs.SketchSpec(sk, 450, 48, **kw), rs.RngStream(9))
    store = dist.HashStore()
    dist.init_process_group("gloo", store=store, rank=0, world_size=1)
    try:
        got = rand_lupp_adaptive_sharded(a, 48, tau, rs.SketchSpec(sk, 450, 48, **kw), rs.RngStream(9))
    finally:
        dist.destroy_process_group()
    assert got.rank == ref.rank and got.status == ref.status and got.rank > 48
    assert np.array_equal(got.row_idx, ref.row_idx)
    assert [(r.k, r.e_schur) for r in got.trace] == [(r.k, r.e_schur) for r in ref.trace]
    assert np.array_equal(got.w, ref.w)


def _worker(rank, world, port, case, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    sys.path[:0] = [REPO, HERE]
    import torch
    import torch.distributed as dist

    import paper_2310_09417_b200 as rs
    from paper_2310_09417_b200.sharded import rand_lupp_adaptive_sharded

    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        m, n, b, taur, seed, counts = case
        a = _matrix(m, n, seed)
        lo = sum(counts[:rank])
        hi = lo + counts[rank]
        tau = taur * np.linalg.norm(a)
        spec = rs.SketchSpec("gaussian", n, b)
        res = rand_lupp_adaptive_sharded(a[lo:hi], b, tau, spec, rs.RngStream(seed + 1))
        q.put((rank, res.rank, np.asarray(res.row_idx), res.status,
               [(r.k, r.e_schur) for r in res.trace], np.asarray(res.w)))
    except Exception as e:
        q.put((rank, "error", repr(e)))
        raise
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("case", [
    (900, 600, 64, 1e-9, 3, [400, 500]),
    (1000, 700, 32, 1e-11, 5, [300, 350, 350]),
    (900, 700, 128, 1e-9, 7, [450, 450]),
    (1000, 800, 96, 1e-11, 8, [200, 500, 300]),
], ids=["w2-b64", "w3-b32", "w2-b128", "w3-b96"])
def test_sharded_multi_rank_one_gpu(case):
    import torch.multiprocessing as mp

    m, n, b, taur, seed, counts = case
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
            item = q.get(timeout=300)
            assert item[1] != "error", item
            outs[item[0]] = item
    finally:
        for p in procs:
            p.join(timeout=60)
            if p.is_alive():
                p.kill()
    a = _matrix(m, n, seed)
    ref = _single(a, b, taur * np.linalg.norm(a), seed + 1)
    w_parts = []
    for r in range(world):
        _, k, row_idx, status, trace, w = outs[r]
        assert k == ref.rank and status == ref.status
        assert np.array_equal(row_idx, ref.row_idx)
        assert [t[0] for t in trace] == [t.k for t in ref.trace]
        assert [t[1] for t in trace] == [t.e_schur for t in ref.trace]  # bit for bit
        w_parts.append(w)
    w = np.vstack(w_parts)
    na = np.linalg.norm(a)
    res = np.linalg.norm(a - w @ a[ref.row_idx]) / na
    res_ref = np.linalg.norm(a - ref.w @ a[ref.row_idx]) / na
    assert res <= 1.5 * res_ref + 1e-13, (res, res_ref)
