"""Host-buffer (pinned) N=16384 multiply end to end: AUTO (streamed DMMA) vs
MODE_OZAKI (B prepared once, A streamed in row panels), plus the bitwise check
of the host Ozaki result against the device-resident Ozaki call."""
import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np
import torch
import paper_1012_2273_b200 as P
ctx = P.Context(0)
n = int(os.environ.get("OZAKI_E2E_N", 16384))
A = ctx.fill(P.DIST_UNIFORM, 0, n, n); B = ctx.fill(P.DIST_UNIFORM, 1, n, n)
a = A.cpu().pin_memory().numpy(); b = B.cpu().pin_memory().numpy()
c = torch.empty((n, n), dtype=torch.float64).pin_memory().numpy()
want = ctx.dgemm(A, B, mode=P.MODE_OZAKI).cpu().numpy()
del A, B
torch.cuda.empty_cache()
for mode_name, mode in (("auto", P.MODE_AUTO), ("ozaki", P.MODE_OZAKI)):
    ts = [ctx.matmul_host(a, b, mode=mode, out=c)[1] for _ in range(3)]
    print(mode_name, [round(t * 1e3, 1) for t in ts], round(2 * n**3 / min(ts) / 1e12, 1), "TFLOP/s e2e")
print("ozaki host == ozaki device (bitwise):", bool((c.view(np.uint64) == want.view(np.uint64)).all()))
