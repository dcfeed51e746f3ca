import sys, numpy as np, torch
import paper_2310_09417_b200 as rs
from paper_2310_09417_b200 import _device
for key in [(3,77),(0,0)]:
    for n in (1000, 5000, 60000, 70000, 100000, 1048576):
        s = rs.RngStream(*key)
        ref = s.generator().standard_normal(n)
        got = _device.gaussian(s, n, 1, unit=True).cpu().numpy().ravel()
        bad = np.flatnonzero(ref != got)
        print(key, n, bad.size, bad[:3], (got[bad[0]], ref[bad[0]]) if bad.size else "")
