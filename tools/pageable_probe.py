"""Host-buffer multiply from pageable vs pinned numpy arrays (the staging ring of
csrc/staging.cu) at N = 2048 / 4096 / 8192, plus single-thread numpy copy speed."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1012_2273_b200 as P
ctx = P.Context(0)
print("cores", len(os.sched_getaffinity(0)))
for n in (2048, 4096, 8192):
    a = np.random.rand(n, n); b = np.random.rand(n, n)
    ap = torch.from_numpy(a).pin_memory().numpy(); bp = torch.from_numpy(b).pin_memory().numpy()
    cp = torch.empty((n, n), dtype=torch.float64).pin_memory().numpy()
    c = np.empty((n, n))
    for name, x, y, z in (("pageable", a, b, c), ("pinned", ap, bp, cp)):
        ts = []
        for _ in range(3):
            _, el = ctx.matmul_host(x, y, out=z)
            ts.append(el)
        print(json.dumps({"n": n, "kind": name, "ms": min(ts) * 1e3, "GBps_io": 24 * n * n / min(ts) / 1e9}), flush=True)
    t0 = time.perf_counter(); d = a.copy(); t1 = time.perf_counter()
    print(json.dumps({"n": n, "numpy_copy_GBps": 8 * n * n / (t1 - t0) / 1e9}))
