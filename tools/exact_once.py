"""Three EXACT multiplies per N (default 500), for ncu captures of the exact kernels:
python tools/exact_once.py 500 1000"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1012_2273_b200 as P  # noqa: E402

ctx = P.Context(0)
for n in [int(x) for x in sys.argv[1:]] or [500]:
    A = ctx.fill(P.DIST_UNIFORM, 0, n, n)
    B = ctx.fill(P.DIST_UNIFORM, 1, n, n)
    C = torch.empty_like(A)
    for _ in range(3):
        ctx.dgemm(A, B, C, mode=P.MODE_EXACT)
    torch.cuda.synchronize()
    print(n, ctx.last_plan, flush=True)
