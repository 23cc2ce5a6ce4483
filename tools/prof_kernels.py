"""One launch of each kernel family (for ncu -k regex:... captures)."""
import sys
import torch
sys.path.insert(0, ".")
import paper_1012_2273_b200 as P

ctx = P.Context(0)
which = sys.argv[1] if len(sys.argv) > 1 else "all"
if which in ("all", "ffma"):
    n = 8192
    A = ctx.fill(P.DIST_NORMAL, 0, n, n, dtype=torch.float32)
    B = ctx.fill(P.DIST_NORMAL, 1, n, n, dtype=torch.float32)
    for _ in range(2):
        ctx.sgemm(A, B)
if which in ("all", "exact"):
    n = 4096
    A = ctx.fill(P.DIST_UNIFORM, 0, n, n)
    B = ctx.fill(P.DIST_UNIFORM, 1, n, n)
    for _ in range(2):
        ctx.dgemm(A, B, mode=P.MODE_EXACT)
if which == "none":
    n = 16384
    A = ctx.fill(P.DIST_UNIFORM, 0, n, n)
    B = ctx.fill(P.DIST_UNIFORM, 1, n, n)
    ctx.dgemm(A, B, mode=P.MODE_DMMA)
if which == "families":
    # one launch per kernel family at its representative size
    n = 8192
    A = ctx.fill(P.DIST_NORMAL, 0, n, n, dtype=torch.float32)
    B = ctx.fill(P.DIST_NORMAL, 1, n, n, dtype=torch.float32)
    ctx.sgemm(A, B)
    del A, B
    n = 4096
    A = ctx.fill(P.DIST_UNIFORM, 0, n, n)
    B = ctx.fill(P.DIST_UNIFORM, 1, n, n)
    ctx.dgemm(A, B, mode=P.MODE_EXACT)
    n = 1000
    A = ctx.fill(P.DIST_UNIFORM, 0, n, n)
    B = ctx.fill(P.DIST_UNIFORM, 1, n, n)
    ctx.dgemm(A, B, mode=P.MODE_AUTO)
    n = 250
    A = ctx.fill(P.DIST_UNIFORM, 0, n, n)
    B = ctx.fill(P.DIST_UNIFORM, 1, n, n)
    ctx.dgemm(A, B, mode=P.MODE_AUTO)
    n = 4099
    A = ctx.fill(P.DIST_INT8, 0, n, n)
    B = ctx.fill(P.DIST_INT8, 1, n, n)
    ctx.dgemm(A, B, mode=P.MODE_AUTO)   # pack_f64_kernel x2 + DMMA
if which == "tiny":
    for n in (10, 64, 250, 500):
        A = ctx.fill(P.DIST_UNIFORM, 0, n, n)
        B = ctx.fill(P.DIST_UNIFORM, 1, n, n)
        for _ in range(2):
            ctx.dgemm(A, B, mode=P.MODE_AUTO)
            ctx.dgemm(A, B, mode=P.MODE_EXACT)
if which in ("all", "small"):
    n = 1000
    A = ctx.fill(P.DIST_UNIFORM, 0, n, n)
    B = ctx.fill(P.DIST_UNIFORM, 1, n, n)
    for _ in range(2):
        ctx.dgemm(A, B, mode=P.MODE_AUTO)
torch.cuda.synchronize()
print("ok")
