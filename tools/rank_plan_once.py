"""Rank 0's multiply of one row-block round at P ranks, on one GPU (for ncu
DRAM-traffic captures of the per-rank plan, profiles/*_ncu_summary*.json).

rowblock.cu gives rank 0 rows [0, N/P) and multiplies them as S = 2
sub-blocks (split_rows of its rows), each a separate launch with the
whole-problem kernel choice; this replays exactly those launches (AUTO fp64
for configs[3], FFMA fp32 for configs[4]).

  python tools/rank_plan_once.py f64 16384 2 4 8
  python tools/rank_plan_once.py f32 32768 1 2 4 8
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1012_2273_b200 as P  # noqa: E402


def main():
    kind, n = sys.argv[1], int(sys.argv[2])
    ps = [int(x) for x in sys.argv[3:]] or [2, 4, 8]
    ctx = P.Context(0)
    f32 = kind == "f32"
    dt = torch.float32 if f32 else torch.float64
    dist = P.DIST_NORMAL if f32 else P.DIST_UNIFORM
    A = ctx.fill(dist, 0, n, n, dtype=dt)
    B = ctx.fill(dist, 1, n, n, dtype=dt)
    C = torch.empty_like(A)
    ctx.tune("MMWS_GPU_NO_STREAMK", "1")  # a distributed round never uses stream-K
    for p in ps:
        rows0 = P.split_rows(n, p)[0][1]
        subs = P.split_rows(rows0, 2) if p > 1 and n // p >= 1024 else [(0, rows0)]
        for off, rows in subs:
            a, c = A[off:off + rows], C[off:off + rows]
            if f32:
                ctx.sgemm(a, B, c, mode=P.MODE_FFMA)
            else:
                ctx.dgemm(a, B, c, mode=P.MODE_AUTO)
        torch.cuda.synchronize()
        print(f"P={p} rows0={rows0} launches={len(subs)} plan={ctx.last_plan}", flush=True)


if __name__ == "__main__":
    main()
