"""One device-pointer multiply per MMWS_GPU_DMMA_PLAN given on the command
line (for ncu: one kernel launch per plan).
PLAN[:G] also sets the raster group (MMWS_GPU_RASTER_GROUP=G).
Usage: python tools/plan_once.py N PLAN[:G] [PLAN[:G] ...]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1012_2273_b200 as P  # noqa: E402

n = int(sys.argv[1])
ctx = P.Context(0)
A = ctx.fill(P.DIST_UNIFORM, 0, n, n)
B = ctx.fill(P.DIST_UNIFORM, 1, n, n)
C = torch.empty_like(A)
for tok in sys.argv[2:]:
    plan, _, group = tok.partition(":")
    ctx.tune("MMWS_GPU_DMMA_PLAN", plan)
    ctx.tune("MMWS_GPU_RASTER_GROUP", group or None)
    ctx.dgemm(A, B, C, mode=P.MODE_DMMA)
    torch.cuda.synchronize()
    print(tok, ctx.last_plan, flush=True)
