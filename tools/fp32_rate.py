"""FP32 FFMA2 multiply rate (TFLOP/s, min of 3 CUDA-event timings) at the given N.
Usage: python tools/fp32_rate.py [N ...]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1012_2273_b200 as P
ctx = P.Context(0)
for n in [int(x) for x in sys.argv[1:]] or (8192, 16384):
    A = ctx.fill(P.DIST_NORMAL, 0, n, n, dtype=torch.float32)
    B = ctx.fill(P.DIST_NORMAL, 1, n, n, dtype=torch.float32)
    C = torch.empty_like(A)
    ctx.sgemm(A, B, C); torch.cuda.synchronize()
    ts = []
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); ctx.sgemm(A, B, C); e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
    print(n, round(2*n**3/min(ts)/1e9, 2))
