"""Two fp32 multiplies at N=4096 (for ncu captures of the FFMA2 kernel)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1012_2273_b200 as P  # noqa: E402

ctx = P.Context(0)
n = 4096
A = ctx.fill(P.DIST_NORMAL, 0, n, n, dtype=torch.float32)
B = ctx.fill(P.DIST_NORMAL, 1, n, n, dtype=torch.float32)
C = torch.empty_like(A)
for _ in range(2):
    ctx.sgemm(A, B, C)
torch.cuda.synchronize()
print("ok")
