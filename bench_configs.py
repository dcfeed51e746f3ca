"""Secondary BASELINE.json configs (bench.py measures configs[1]).

  python bench_configs.py [--cpu]   -> one JSON line per config

cfg1  column_id of a 4096^2 fp64 fast-decay matrix, k = 256, seed 0
cfg3  adaptive CUR of a 32768 x 16384 fp32 nonnegative low-rank(200)+noise
      matrix, b = 64, tau = 1e-5 ||A||_F (relative; absolute 1e-5 is below the
      fp32 floor)
cfg4  column_id / rand_lupp of the Kahan 16384^2 matrix (zeta 0.99), k = 1024
cfg5  adaptive column ID of the 65536^2 randomized-Hadamard fast-decay matrix at 1 GPU

GPU times are CUDA-event times with A resident on the device (median of 3
after a warm-up) and end-to-end times through the numpy API.  --cpu adds the
oracle (reference algorithm, numpy/OpenBLAS, all host cores) on the same
inputs.
"""

import json
import os
import sys
import time

import numpy as np
import torch

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)
sys.path.insert(0, os.path.join(REPO, "oracle"))

import paper_2310_09417_b200 as rs  # noqa: E402
from bench import FP64_DMMA_PEAK_TFLOPS, algo_flops, gen_fast_decay_device  # noqa: E402


def dev_time(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        out = fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return float(np.median(ts)), out


def wall(fn, reps=1):
    ts = []
    out = None
    for _ in range(reps):
        t0 = time.perf_counter()
        out = fn()
        ts.append(time.perf_counter() - t0)
    return float(np.median(ts)), out


def cpu_run(fn):
    from threadpoolctl import threadpool_limits

    with threadpool_limits(limits=os.cpu_count()):
        return wall(fn)


def cfg1(do_cpu):
    import randskel_oracle as orc

    n, k = 4096, 256
    a = gen_fast_decay_device(n, 1e-16, 0, "cuda")
    spec = rs.SketchSpec("gaussian", n, k)
    ms, r = dev_time(lambda: rs.column_id(a, k, spec, rs.RngStream(0)), reps=5)
    ah = a.cpu().numpy()
    wall(lambda: rs.column_id(ah, k, spec, rs.RngStream(0)))  # first call: host staging buffers, module loads
    e2e, _ = wall(lambda: rs.column_id(ah, k, spec, rs.RngStream(0)), reps=5)
    f = algo_flops(n, n, k, 0)
    line = {"config": "cfg1 column_id 4096^2 fp64 fast-decay k=256", "gpu_ms": ms, "e2e_ms": 1e3 * e2e,
            "tflops": f / ms / 1e9, "frac_fp64_dmma": f / ms / 1e9 / FP64_DMMA_PEAK_TFLOPS}
    if do_cpu:
        t, (cidx, x) = cpu_run(lambda: orc.column_id(ah, k, 0))
        line.update(cpu_s=t, cpu_cores=os.cpu_count(), speedup_e2e=t / e2e,
                    col_idx_equal=bool(np.array_equal(np.asarray(r.col_idx.cpu()), cidx)))
    return line


def cfg3(do_cpu):
    import randskel_oracle as orc

    m, n, r0, b = 32768, 16384, 200, 64
    a32 = rs.gen_nonneg_lowrank(m, n, r0, 1e-6, rs.RngStream(0).child(1 << 41))
    na = float(torch.linalg.norm(a32.double()))
    tau = 1e-5 * na
    spec = rs.SketchSpec("gaussian", n, b)
    ms, (cur, res) = dev_time(lambda: rs.cur_decompose_adaptive(a32, b, tau, spec, rs.RngStream(0)), reps=2)
    ah = a32.cpu().numpy()
    wall(lambda: rs.cur_decompose_adaptive(ah, b, tau, spec, rs.RngStream(0)))  # first call
    e2e, _ = wall(lambda: rs.cur_decompose_adaptive(ah, b, tau, spec, rs.RngStream(0)), reps=3)
    k = res.rank
    # ID flops with rows as candidates + CUR linking solves (2 m n k + 2 m k^2 ...)
    f = algo_flops(m, n, k, b) + 2.0 * m * n * k + 2.0 * m * k * k
    line = {"config": "cfg3 adaptive CUR 32768x16384 fp32 (computed in fp64) b=64 tau=1e-5||A||",
            "rank": k, "status": res.status, "cur_status": cur.status, "gpu_ms": ms,
            "e2e_ms": 1e3 * e2e, "tflops": f / ms / 1e9}
    if do_cpu:
        a64 = ah.astype(np.float64)
        t, out = cpu_run(lambda: orc.cur_from_rows(
            a64, orc.rand_lupp_adaptive(a64, b, tau, 0, want_w=False)["row_idx"], k))
        line.update(cpu_s=t, cpu_cores=os.cpu_count(), speedup_e2e=t / e2e)
    return line


def cfg4(do_cpu):
    import randskel_oracle as orc

    n, k = 16384, 1024
    a = torch.as_tensor(orc.gen_kahan(n, 0.99)).cuda()
    spec = rs.SketchSpec("gaussian", n, k)
    ms, r = dev_time(lambda: rs.column_id(a, k, spec, rs.RngStream(0)), reps=5)
    ah = a.cpu().numpy()
    wall(lambda: rs.column_id(ah, k, spec, rs.RngStream(0)))  # first call: host staging buffers, module loads
    e2e, _ = wall(lambda: rs.column_id(ah, k, spec, rs.RngStream(0)), reps=3)
    f = algo_flops(n, n, k, 0)
    line = {"config": "cfg4 column_id Kahan 16384^2 fp64 k=1024", "gpu_ms": ms, "e2e_ms": 1e3 * e2e,
            "tflops": f / ms / 1e9, "frac_fp64_dmma": f / ms / 1e9 / FP64_DMMA_PEAK_TFLOPS}
    if do_cpu:
        t, (cidx, x) = cpu_run(lambda: orc.column_id(ah, k, 0))
        ov = len(set(np.asarray(r.col_idx.cpu()).tolist()) & set(cidx.tolist()))
        line.update(cpu_s=t, cpu_cores=os.cpu_count(), speedup_e2e=t / e2e,
                    col_idx_equal=bool(np.array_equal(np.asarray(r.col_idx.cpu()), cidx)), overlap=ov)
    return line


def cfg5(do_cpu):
    """cfg5 at one GPU (the sharded form runs this loop split over ranks):
    adaptive column ID of a 65536^2 fp64 fast-decay matrix, b=64, tau=1e-8."""
    n, b, tau = int(os.environ.get("CFG5_N", 65536)), 64, 1e-8
    a, _ = rs.gen_fast_decay_hadamard(n, 1e-16, rs.RngStream(0).child(1 << 41))
    torch.cuda.synchronize()
    spec = rs.SketchSpec("gaussian", n, b)
    ms, res = dev_time(lambda: rs.rand_lupp_adaptive(a.T, b, tau, spec, rs.RngStream(0)), reps=1)
    k = res.rank
    f = algo_flops(n, n, k, b)
    line = {"config": f"cfg5 adaptive column ID {n}^2 fp64 fast-decay (Hadamard bases) b=64 tau=1e-8, 1 GPU",
            "rank": k, "status": res.status, "blocks": len(res.trace) + 1, "gpu_ms": ms,
            "tflops": f / ms / 1e9, "frac_fp64_dmma": f / ms / 1e9 / FP64_DMMA_PEAK_TFLOPS,
            "cpu": "infeasible here (SURVEY 8d: ~2-4 h on the host cores)"}
    del res
    return line


if __name__ == "__main__":
    do_cpu = "--cpu" in sys.argv
    which = [a for a in sys.argv[1:] if a.startswith("cfg")] or ["cfg1", "cfg3", "cfg4"]
    for name in which:
        print(json.dumps(globals()[name](do_cpu)), flush=True)
