"""EXACT-mode (bitwise matmul_seq) multiply rate (TFLOP/s, min of 3 CUDA-event
timings) at the given N, with a sha256 of a ragged product (ring-geometry and
other rebuilds must keep the bits).  Usage: python tools/exact_rate.py [N ...]"""
import hashlib
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1012_2273_b200 as P

ctx = P.Context(0)
A = ctx.fill(P.DIST_UNIFORM, 0, 1031, 777)
B = ctx.fill(P.DIST_UNIFORM, 1, 777, 1283)
C = ctx.dgemm(A, B, mode=P.MODE_EXACT)
torch.cuda.synchronize()
print("sha", hashlib.sha256(C.cpu().numpy().tobytes()).hexdigest()[:16], ctx.last_plan)
for n in [int(x) for x in sys.argv[1:]] or (2048, 4096, 8192):
    A = ctx.fill(P.DIST_UNIFORM, 0, n, n)
    B = ctx.fill(P.DIST_UNIFORM, 1, n, n)
    C = torch.empty_like(A)
    ctx.dgemm(A, B, C, mode=P.MODE_EXACT)
    torch.cuda.synchronize()
    ts = []
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        ctx.dgemm(A, B, C, mode=P.MODE_EXACT)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    print("N", n, round(2 * n ** 3 / min(ts) / 1e9, 2), "TFLOP/s", ctx.last_plan)
