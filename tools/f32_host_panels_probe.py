"""configs[4] through the host entry (pinned fp32 A, B, C, N=32768 by default)
against the number of row panels (MMWS_GPU_HOST_PANELS, 0 = built-in rule):
host wall clock per call.  Usage: python tools/f32_host_panels_probe.py [N] [panels ...]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_1012_2273_b200 as P

ctx = P.Context(0)
n = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
arms = [int(x) for x in sys.argv[2:]] or [0, 8, 12, 16, 24, 32]
A = ctx.fill(P.DIST_NORMAL, 0, n, n, dtype=torch.float32)
B = ctx.fill(P.DIST_NORMAL, 1, n, n, dtype=torch.float32)
hA = torch.empty((n, n), dtype=torch.float32, pin_memory=True)
hB = torch.empty((n, n), dtype=torch.float32, pin_memory=True)
hC = torch.empty((n, n), dtype=torch.float32, pin_memory=True)
hA.copy_(A)
hB.copy_(B)
del A, B
torch.cuda.empty_cache()
a, b, c = hA.numpy(), hB.numpy(), hC.numpy()
for p in arms:
    ctx.tune("MMWS_GPU_HOST_PANELS", str(p) if p else None)
    ctx.master_run_host(a, b, c, mode=P.MODE_FFMA)
    ts = []
    for _ in range(2):
        t0 = time.perf_counter()
        ctx.master_run_host(a, b, c, mode=P.MODE_FFMA)
        ts.append(time.perf_counter() - t0)
    print(f"panels {p or 'rule'}: {min(ts) * 1e3:.1f} ms  {2.0 * n ** 3 / min(ts) / 1e12:.2f} TFLOP/s", flush=True)
