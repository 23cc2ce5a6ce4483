"""Host-entry wall time (min / median of 50) for small pageable multiplies."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1012_2273_b200 as P
ctx = P.Context(0)
for n in (100, 250, 500):
    a = np.random.rand(n, n); b = np.random.rand(n, n)
    for _ in range(5): ctx.matmul_host(a, b)
    ts = sorted(ctx.matmul_host(a, b)[1] for _ in range(50))
    print(n, round(ts[0]*1e6,1), round(ts[25]*1e6,1))
