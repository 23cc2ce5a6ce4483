"""Small runs of every kernel family and host path (a quick exerciser; compute-sanitizer
is closed on this pool, so out-of-bounds writes are guarded by the canary test
tests/test_gpu_parity.py::test_no_writes_outside_c instead)."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_1012_2273_b200 as P

ctx = P.Context(0)
for (m, k, n) in [(1, 1, 1), (7, 3, 5), (130, 129, 131), (257, 300, 129), (300, 64, 700)]:
    A = ctx.fill(P.DIST_UNIFORM, 1, m, k)
    B = ctx.fill(P.DIST_UNIFORM, 2, k, n)
    for mode in (P.MODE_AUTO, P.MODE_EXACT, P.MODE_DMMA, P.MODE_DMMA_SMALL):
        ctx.dgemm(A, B, mode=mode)
    Af = ctx.fill(P.DIST_NORMAL, 1, m, k, dtype=torch.float32)
    Bf = ctx.fill(P.DIST_NORMAL, 2, k, n, dtype=torch.float32)
    ctx.sgemm(Af, Bf)
    ctx.sgemm(Af[:, :k - 1] if k > 1 else Af, Bf[:k - 1] if k > 1 else Bf)
big = ctx.fill(P.DIST_UNIFORM, 3, 301, 303)
ctx.dgemm(big[1:200, 1:300], big[:299, 2:150], mode=P.MODE_DMMA)
ctx.dgemm(big[1:200, 1:300], big[:299, 2:150], mode=P.MODE_EXACT)
a = np.random.rand(2304, 512)
b = np.random.rand(512, 2304)
ctx.matmul_host(a, b)                     # streamed persistent kernel
ctx.matmul_host(a[:1300], b[:, :1300].copy())
g = ctx.graph_dgemm(A, B, torch.empty((m, n), dtype=torch.float64, device="cuda"))
g.launch()
torch.cuda.synchronize()
print("exercise ok", ctx.launches)
