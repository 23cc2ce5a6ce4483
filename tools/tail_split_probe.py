"""Wave-tail experiment: one AUTO multiply vs the same C computed as two row
ranges (a whole number of 32x32-tile waves + the remainder, which AUTO
puts on 16x16 tiles), launched back to back; device time per call (CUDA
events around 20 calls), bits compared."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_1012_2273_b200 as P

ctx = P.Context(0)
s = torch.cuda.current_stream()  # ctx.dgemm launches on the caller's current stream


def dev_us(fn, reps=10, inner=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(reps):
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        torch.cuda._sleep(int(inner * 80e-6 * 2e9))
        e0.record(s)
        for _ in range(inner):
            fn()
        e1.record(s)
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1) * 1e3 / inner)
    return best


for n in [int(x) for x in sys.argv[1:]] or [500, 750, 1000, 1250, 1500]:
    A = ctx.fill(P.DIST_UNIFORM, 0, n, n)
    B = ctx.fill(P.DIST_UNIFORM, 1, n, n)
    C = torch.empty_like(A)
    C2 = torch.empty_like(A)
    t1 = dev_us(lambda: ctx.dgemm(A, B, C))
    plan = ctx.last_plan
    tiles_n = (n + 31) // 32
    res = {"n": n, "one_launch_us": round(t1, 2), "plan": plan}
    for slots in (6, 5, 4):
        # rows covered by whole waves of `slots` 32x32 tiles per SM
        full = (148 * slots // tiles_n) * 32
        for waves in (1, 2, 3):
            m1 = min(n, full * waves)
            if m1 >= n or m1 <= 0:
                continue

            def two():
                ctx.dgemm(A[:m1], B, C2[:m1])
                ctx.dgemm(A[m1:], B, C2[m1:])
            t2 = dev_us(two)
            same = bool(torch.equal(C.view(torch.int64), C2.view(torch.int64)))
            res[f"split_s{slots}_w{waves}"] = [m1, round(t2, 2), same]
    print(json.dumps(res), flush=True)
