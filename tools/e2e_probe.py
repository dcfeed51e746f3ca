"""Where does end-to-end (host numpy in/out) time go?  PYTHONPATH=. python tools/e2e_probe.py"""
import time

import numpy as np
import torch

import paper_2310_09417_b200 as rs
from paper_2310_09417_b200 import _device

n = 20000
dev = torch.device("cuda")
a_pin = torch.empty((n, n), dtype=torch.float64, pin_memory=True)
a_pin.normal_()
a_np = a_pin.numpy()
a_page = np.empty((n, n))
a_page[:] = a_np


def t(fn, label):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    out = fn()
    torch.cuda.synchronize()
    print(f"{label}: {1e3 * (time.perf_counter() - t0):.1f} ms")
    return out


for _ in range(2):
    m = t(lambda: _device.as_matrix(a_np.T), "as_matrix(pinned numpy .T)")
    del m
    m = t(lambda: _device.as_matrix(a_page.T), "as_matrix(pageable numpy .T)")
    del m
    w = torch.randn(n, 14500, dtype=torch.float64, device=dev)
    h = t(lambda: _device.to_output(w, "numpy"), "to_output(W 20000x14500) -> numpy (pinned path)")
    del h
    h = t(lambda: w.cpu().numpy(), "W.cpu().numpy() (pageable)")
    del h
    hp = np.empty((n, 14500))
    ht = torch.from_numpy(hp)
    t(lambda: ht.copy_(w), "copy_ into preallocated pageable numpy")
    del w, hp, ht
