"""Normwise errors of each path against the fp64 oracle on sampled rows
(development aid; the pass/fail bounds live in tests/test_gpu_parity.py)."""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import oracle as O  # noqa: E402
import paper_1012_2273_b200 as P  # noqa: E402


def nw(x, r):
    return float(np.linalg.norm(x - r) / np.linalg.norm(r))


ctx = P.Context(0)
out = {}
n = 32768
A = ctx.fill(P.DIST_NORMAL, 0, n, n, dtype=torch.float32)
B = ctx.fill(P.DIST_NORMAL, 1, n, n, dtype=torch.float32)
rows = [0, 1, 4095, 4096, 16383, 16384, 24575, 32767]
C = ctx.sgemm(A, B)
torch.cuda.synchronize()
want = O.matmul_rows(list(range(len(rows))), A[rows].cpu().numpy(), B.cpu().numpy())
got = C[rows].cpu().numpy().astype(np.float64)
out["c5_fp32_n32768_normwise"] = nw(got, want)
# single-chain fp32 reference point: plain fp32 dot products in ascending k (numpy float32 accumulate)
a32, b32 = A[rows[:2]].cpu().numpy(), B.cpu().numpy()
seq = np.zeros((2, n), dtype=np.float32)
for kk in range(n):
    seq += a32[:, kk:kk + 1] * b32[kk]
out["single_chain_fp32_2rows_normwise"] = nw(seq.astype(np.float64), want[:2])
del A, B, C
n = 16384
A = ctx.fill(P.DIST_UNIFORM, 0, n, n)
B = ctx.fill(P.DIST_UNIFORM, 1, n, n)
rows = [0, 1, 2047, 2048, 4095, 8191, 12288, 16383]
want = O.matmul_rows(list(range(len(rows))), A[rows].cpu().numpy(), B.cpu().numpy())
out["c4_dmma_n16384_normwise"] = nw(ctx.dgemm(A, B)[rows].cpu().numpy(), want)
print(json.dumps(out))
