"""Timeline of the streamed host-buffer multiply (MMWS_GPU_PIPELINE_TRACE=1):
H2D end, kernel start/end and D2H end relative to the first copy, per call.
Usage: MMWS_GPU_PIPELINE_TRACE=1 python tools/pipeline_trace.py [N] [calls]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1012_2273_b200 as P  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
calls = int(sys.argv[2]) if len(sys.argv) > 2 else 3
ctx = P.Context(0)
A = ctx.fill(P.DIST_UNIFORM, 0, n, n)
B = ctx.fill(P.DIST_UNIFORM, 1, n, n)
a = A.cpu().pin_memory().numpy()
b = B.cpu().pin_memory().numpy()
c = torch.empty((n, n), dtype=torch.float64).pin_memory().numpy()
C = ctx.dgemm(A, B)
torch.cuda.synchronize()
for _ in range(3):                       # device-resident multiply for comparison
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    ctx.dgemm(A, B, C)
    e1.record()
    torch.cuda.synchronize()
    print(f"device dgemm: {e0.elapsed_time(e1):.3f} ms", flush=True)
for _ in range(calls):
    _, el = ctx.master_run_host(a, b, c)
    print(f"call: {el * 1e3:.3f} ms", flush=True)
