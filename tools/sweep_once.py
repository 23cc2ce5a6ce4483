"""Three AUTO fp64 multiplies per N (default: the paper's mid sizes), for ncu
captures of the small-N kernels:  python tools/sweep_once.py 250 500 1000"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1012_2273_b200 as P  # noqa: E402

ctx = P.Context(0)
for n in [int(x) for x in sys.argv[1:]] or [250, 500, 1000]:
    A = ctx.fill(P.DIST_UNIFORM, 0, n, n)
    B = ctx.fill(P.DIST_UNIFORM, 1, n, n)
    C = torch.empty_like(A)
    for _ in range(3):
        ctx.dgemm(A, B, C)
    torch.cuda.synchronize()
    print(n, ctx.last_plan, flush=True)
