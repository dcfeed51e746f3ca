"""cuBLAS DGEMM on the sketch shape, for ncu (learn its tiling).
   ncu --set full -k regex:gemm -c 1 python tools/prof_cublas.py"""
import torch

n = 20000
a = torch.randn(n, n, dtype=torch.float64, device="cuda")
om = torch.randn(n, 64, dtype=torch.float64, device="cuda")
for _ in range(3):
    y = a.T @ om
torch.cuda.synchronize()
print("ok")
