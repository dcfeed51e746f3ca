#!/bin/bash
# One-off GPU box probe: host cores, GPU, DMMA peak, cuBLAS DGEMM, H2D bandwidth, host RNG rate.
mkdir -p gpurun_out
{
nproc; lscpu | grep -E "Model name|Socket|Core|Thread|NUMA node"; free -g | head -2
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv
./tools/dmma_peak
python - <<'PY'
import torch, time, numpy as np, os
from concurrent.futures import ThreadPoolExecutor
d = torch.device("cuda")
for n in (4096, 8192, 16384):
    a = torch.randn(n, n, dtype=torch.float64, device=d); b = torch.randn(n, n, dtype=torch.float64, device=d)
    for _ in range(2): a @ b
    torch.cuda.synchronize(); e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(); r = 5
    for _ in range(r): a @ b
    e1.record(); torch.cuda.synchronize(); ms = e0.elapsed_time(e1) / r
    print(f"cublas dgemm n={n}: {2*n**3/ms/1e9:.1f} TF/s")
m, k = 20000, 64
a = torch.randn(m, m, dtype=torch.float64, device=d); b = torch.randn(m, k, dtype=torch.float64, device=d)
for _ in range(2): a.T @ b
torch.cuda.synchronize(); e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(5): a.T @ b
e1.record(); torch.cuda.synchronize(); ms = e0.elapsed_time(e1) / 5
print(f"cublas dgemm 20000x20000^T x 64: {ms:.3f} ms {2*m*m*k/ms/1e9:.1f} TF/s")
h = torch.empty(256 << 20, dtype=torch.uint8).pin_memory(); g = torch.empty_like(h, device=d)
for _ in range(2): g.copy_(h, non_blocking=True)
torch.cuda.synchronize(); t = time.perf_counter()
for _ in range(5): g.copy_(h, non_blocking=True)
torch.cuda.synchronize(); print(f"H2D pinned {5*h.numel()/(time.perf_counter()-t)/1e9:.1f} GB/s")
t = time.perf_counter()
for _ in range(5): h.copy_(g, non_blocking=True)
torch.cuda.synchronize(); print(f"D2H pinned {5*h.numel()/(time.perf_counter()-t)/1e9:.1f} GB/s")
def draw(i):
    g = np.random.Generator(np.random.Philox(key=[0, i])); return g.standard_normal((20000, 64))
t = time.perf_counter(); [draw(i) for i in range(20)]; dt = time.perf_counter() - t
print(f"host normals 1 thread: {20*20000*64/dt/1e6:.0f} M/s")
nt = os.cpu_count()
with ThreadPoolExecutor(nt) as ex:
    t = time.perf_counter(); list(ex.map(draw, range(8 * nt))); dt = time.perf_counter() - t
print(f"host normals {nt} threads: {8*nt*20000*64/dt/1e6:.0f} M/s")
import numpy; numpy.show_config()
PY
} > gpurun_out/probe.log 2>&1
