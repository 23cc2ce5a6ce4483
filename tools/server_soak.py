"""Soak of the resident latency server (csrc/server.cu): many random tiny
requests (shapes up to 96, AUTO / EXACT, solo-CTA and grid-wide sizes),
interleaved with stream-ordered device calls and host-buffer calls the server
does not take; every result bitwise its precomputed device-entry product.

    python tools/server_soak.py [requests] [seed]
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1012_2273_b200 as P

requests = int(sys.argv[1]) if len(sys.argv) > 1 else 20000
seed = int(sys.argv[2]) if len(sys.argv) > 2 else 1
rng = np.random.default_rng(seed)
ctx = P.Context(0)
cases = []
for i in range(64):
    m, k, n = (int(v) for v in rng.integers(1, 97, size=3))
    a = ctx.fill(P.DIST_UNIFORM, 10 + i, m, k)
    b = ctx.fill(P.DIST_UNIFORM, 500 + i, k, n)
    want = {mode: ctx.dgemm(a, b, mode=mode).cpu().numpy().view(np.uint64).copy()
            for mode in (P.MODE_AUTO, P.MODE_EXACT)}
    cases.append((a.cpu().numpy(), b.cpu().numpy(), a, b, want))
big = ctx.fill(P.DIST_UNIFORM, 9, 300, 300)
big_want = ctx.dgemm(big, big, mode=P.MODE_EXACT).cpu().numpy().view(np.uint64).copy()
torch.cuda.synchronize()
ctx.server_start()
bad = []
t0 = time.perf_counter()
for r in range(requests):
    i = int(rng.integers(0, len(cases)))
    a, b, A, B, want = cases[i]
    mode = P.MODE_AUTO if rng.random() < 0.5 else P.MODE_EXACT
    got, _ = ctx.server_matmul(a, b, mode=mode)
    if not np.array_equal(got.view(np.uint64), want[mode]):
        bad.append((r, i, mode))
    x = rng.random()
    if x < 0.01:     # a stream-ordered device call of the same context
        s = ctx.dgemm(A, B, mode=mode, stream=ctx.stream)
        c = torch.empty_like(s)
        c.copy_(s)
    elif x < 0.02:   # a host-buffer call the server does not take (300 > 96)
        h, _ = ctx.matmul_host(big.cpu().numpy(), big.cpu().numpy(), mode=P.MODE_EXACT)
        if not np.array_equal(h.view(np.uint64), big_want):
            bad.append((r, "host", 300))
dt = time.perf_counter() - t0
ctx.server_stop()
print(json.dumps({"requests": requests, "seed": seed, "seconds": dt, "us_per_request": dt / requests * 1e6,
                  "mismatches": len(bad), "first": bad[:10]}))
sys.exit(1 if bad else 0)
