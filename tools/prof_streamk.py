"""One stream-K DMMA launch (N=2048) and one stream-K exact launch (N=2304),
for ncu: ncu --set full -k regex:"dgemm_(dmma|exact)" -c 2 python tools/prof_streamk.py"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1012_2273_b200 as P  # noqa: E402

ctx = P.Context(0)
for n, mode in ((2048, P.MODE_AUTO), (2304, P.MODE_EXACT)):
    A = ctx.fill(P.DIST_UNIFORM, 0, n, n)
    B = ctx.fill(P.DIST_UNIFORM, 1, n, n)
    C = ctx.dgemm(A, B, mode=mode)
torch.cuda.synchronize()
print("ok")
