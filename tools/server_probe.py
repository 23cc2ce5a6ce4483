"""Latency-server wall time per call (min / median) for N in {10..96} and several
grid sizes.  Usage: python tools/server_probe.py [CTAS ...]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1012_2273_b200 as P
ctx = P.Context(0)
for ctas in [int(x) for x in (sys.argv[1:] or [1, 2, 4, 8, 16, 32])]:
    os.environ["MMWS_GPU_SERVER_CTAS"] = str(ctas)
    ctx.server_start()
    row = {"ctas": ctas}
    for n in (10, 24, 32, 50, 64, 96):
        a = np.random.rand(n, n); b = np.random.rand(n, n)
        for _ in range(20): ctx.server_matmul(a, b)
        ts = sorted(ctx.server_matmul(a, b)[1] for _ in range(300))
        row[n] = round(ts[0] * 1e6, 2), round(ts[150] * 1e6, 2)
    ctx.server_stop()
    print(json.dumps(row), flush=True)
