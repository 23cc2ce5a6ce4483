"""EXACT-mode device time per call for mid-size and panel shapes (CUDA events
around back-to-back calls on the caller's stream) and a sha256 of C, so runs
with different plan settings can be compared for speed and bits."""
import hashlib
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_1012_2273_b200 as P

ctx = P.Context(0)
s = torch.cuda.current_stream()
shapes = [(int(x), int(x), int(x)) for x in sys.argv[1:]] or [(336, 336, 336), (400, 400, 400), (500, 500, 500), (640, 640, 640), (700, 700, 700),
          (800, 800, 800), (128, 500, 500), (128, 1000, 1000), (256, 1000, 1000),
          (1000, 1000, 1000), (256, 2000, 2000)]
for (m, k, n) in shapes:
    A = ctx.fill(P.DIST_UNIFORM, 0, m, k)
    B = ctx.fill(P.DIST_UNIFORM, 1, k, n)
    C = torch.empty((m, n), dtype=torch.float64, device="cuda")
    for _ in range(3):
        ctx.dgemm(A, B, C, mode=P.MODE_EXACT)
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(10):
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        torch.cuda._sleep(int(20 * 100e-6 * 2e9))
        e0.record(s)
        for _ in range(20):
            ctx.dgemm(A, B, C, mode=P.MODE_EXACT)
        e1.record(s)
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1) * 1e3 / 20)
    sha = hashlib.sha256(C.cpu().numpy().tobytes()).hexdigest()[:16]
    print(json.dumps({"xp": os.environ.get("XP_EXACT32", "0"), "shape": [m, k, n],
                      "us": round(best, 2), "tflops": round(2.0 * m * n * k / best / 1e6, 2),
                      "plan": ctx.last_plan, "sha": sha}), flush=True)
