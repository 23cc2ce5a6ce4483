"""Small runs of the round-2 code paths (fp32 packing, per-graph workspace,
1-rank NCCL world with both gathers and the progress board, narrow host-pipeline
tail) for compute-sanitizer --tool memcheck."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1012_2273_b200 as P
ctx = P.Context(0)
# fp32 packing path, unaligned
big_a = ctx.fill(P.DIST_NORMAL, 5, 61, 131, dtype=torch.float32)
big_b = ctx.fill(P.DIST_NORMAL, 6, 130, 77, dtype=torch.float32)
ctx.sgemm(big_a[1:60, 3:130], big_b[1:128, 1:76]); torch.cuda.synchronize()
# graph with its own workspace + regrow
big = ctx.fill(P.DIST_UNIFORM, 51, 101, 103)
A = big[:, 1:100]; B = ctx.fill(P.DIST_UNIFORM, 52, 99, 97)
C = torch.empty((101, 97), dtype=torch.float64, device="cuda")
g = ctx.graph_dgemm(A, B, C); g.launch()
big2 = ctx.fill(P.DIST_UNIFORM, 53, 301, 303); ctx.dgemm(big2[:, 1:302], big2[:301, 2:303])
g.launch(); torch.cuda.synchronize(); g.close()
# 1-rank world: both gathers, board marks
ctx.comm_init(1, 0, P.nccl_unique_id())
for knob in (None, "1"):
    ctx.tune("MMWS_GPU_NCCL_GATHER", knob)
    A = ctx.fill(P.DIST_UNIFORM, 0, 130, 70); B = ctx.fill(P.DIST_UNIFORM, 1, 70, 90)
    C = torch.empty((130, 90), dtype=torch.float64, device="cuda")
    ctx.rowblock(130, 90, 70, A, B, C)
a = A.cpu().numpy(); b = B.cpu().numpy()
ctx.master_run_host(a, b)
ctx.comm_destroy()
# host pipeline narrow tail (pinned)
a = torch.from_numpy(np.random.rand(1060, 96)).pin_memory().numpy()
b = torch.from_numpy(np.random.rand(96, 1060)).pin_memory().numpy()
ctx.matmul_host(a, b)
print("memcheck cases ok")
