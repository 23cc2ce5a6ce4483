"""One MODE_OZAKI multiply at N (default 16384) after a warm-up, for the ncu
launch list: ncu --metrics gpu__time_duration.sum -k regex:"exponent|residue|igemm|crt" ..."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1012_2273_b200 as P  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
ctx = P.Context(0)
A = ctx.fill(P.DIST_UNIFORM, 0, n, n)
B = ctx.fill(P.DIST_UNIFORM, 1, n, n)
C = ctx.dgemm(A, B, mode=P.MODE_OZAKI)
torch.cuda.synchronize()
print("ok")
