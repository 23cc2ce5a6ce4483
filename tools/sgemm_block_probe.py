"""fp32 kernel with A staged as it lies (MMWS_GPU_SGEMM_AT=0) or transposed and
staged k-major (=1; unset: the size rule): rate at the given N and a sha256 of
two ragged products (both stagings, and any rebuild with other ring geometries,
must give the same bits).  Run once per value of the knob.
Usage: MMWS_GPU_SGEMM_AT=1 python tools/sgemm_block_probe.py [N ...]"""
import hashlib
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1012_2273_b200 as P

ctx = P.Context(0)
ri = os.environ.get("MMWS_GPU_SGEMM_AT", "default")
for m, k, n in ((2049, 3001, 1537), (333, 5000, 260)):
    A = ctx.fill(P.DIST_NORMAL, 0, m, k, dtype=torch.float32)
    B = ctx.fill(P.DIST_NORMAL, 1, k, n, dtype=torch.float32)
    C = ctx.sgemm(A, B)
    torch.cuda.synchronize()
    print("AT", ri, (m, k, n), hashlib.sha256(C.cpu().numpy().tobytes()).hexdigest()[:16])
for n in [int(x) for x in sys.argv[1:]] or (8192, 16384):
    A = ctx.fill(P.DIST_NORMAL, 0, n, n, dtype=torch.float32)
    B = ctx.fill(P.DIST_NORMAL, 1, n, n, dtype=torch.float32)
    C = torch.empty_like(A)
    ctx.sgemm(A, B, C)
    torch.cuda.synchronize()
    ts = []
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        ctx.sgemm(A, B, C)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    print("AT", ri, "N", n, round(2 * n ** 3 / min(ts) / 1e9, 1), "TFLOP/s")
