"""Spectrum check of the cfg5 Hadamard-basis generator at a small size."""
import torch

from bench_configs import gen_fast_decay_hadamard

n = 1024
a = gen_fast_decay_hadamard(n, 1e-6, 3)
s = torch.linalg.svdvals(a)
d = 1e-6 ** (torch.arange(n, dtype=torch.float64, device="cuda") / (n - 1))
print("max rel sv error", float(((s - d) / d).abs().max()))
