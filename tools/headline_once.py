"""Two launches of the headline multiply (configs[3]: N=16384 fp64 AUTO) and
of the configs[4] fp32 kernel at N=16384, for `ncu --set full -s ... -c 1`
captures of the dominant kernels (launch list: fill x2, dgemm x2, fill x2,
sgemm x2)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1012_2273_b200 as P  # noqa: E402

ctx = P.Context(0)
n = 16384
A = ctx.fill(P.DIST_UNIFORM, 0, n, n)
B = ctx.fill(P.DIST_UNIFORM, 1, n, n)
C = torch.empty_like(A)
for _ in range(2):
    ctx.dgemm(A, B, C)
print(ctx.last_plan, flush=True)
del A, B, C
Af = ctx.fill(P.DIST_NORMAL, 0, n, n, dtype=torch.float32)
Bf = ctx.fill(P.DIST_NORMAL, 1, n, n, dtype=torch.float32)
Cf = torch.empty_like(Af)
for _ in range(2):
    ctx.sgemm(Af, Bf, Cf)
torch.cuda.synchronize()
print(ctx.last_plan, flush=True)
