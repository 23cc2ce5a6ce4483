"""Host-buffer multiply (pageable and pinned) against the number of row
panels (MMWS_GPU_HOST_PANELS, 0 = the built-in rule): interleaved calls,
host wall clock, min / median; bits compared across panel counts."""
import json
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1012_2273_b200 as P

ctx = P.Context(0)
ns = [int(x) for x in sys.argv[1:]] or [500, 750, 1000, 1250, 1500, 2000, 3000]
arms = [0, 1, 2, 3, 4, 8]
for kind in ("pageable", "pinned"):
    for n in ns:
        a = np.random.rand(n, n); b = np.random.rand(n, n); c = np.empty((n, n))
        if kind == "pinned":
            a = torch.from_numpy(a).pin_memory().numpy(); b = torch.from_numpy(b).pin_memory().numpy()
            c = torch.empty((n, n), dtype=torch.float64).pin_memory().numpy()
        ts = {p: [] for p in arms}
        ref = None
        same = True
        for p in arms:
            ctx.tune("MMWS_GPU_HOST_PANELS", str(p))
            for _ in range(3):
                ctx.matmul_host(a, b, out=c)
            if ref is None:
                ref = c.copy()
            same &= bool(np.array_equal(ref, c))
        for _ in range(20 if n <= 2000 else 6):
            for p in arms:
                ctx.tune("MMWS_GPU_HOST_PANELS", str(p))
                t0 = time.perf_counter()
                ctx.matmul_host(a, b, out=c)
                ts[p].append(time.perf_counter() - t0)
        print(json.dumps({"kind": kind, "n": n, "bitwise_same": same,
                          **{f"p{p}": [round(min(v) * 1e6, 1), round(statistics.median(v) * 1e6, 1)]
                             for p, v in ts.items()}}), flush=True)
