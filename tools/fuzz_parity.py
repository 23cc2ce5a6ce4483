"""Time-boxed randomized parity sweep against the CPU oracle (test
infrastructure, like tests/): random shapes (1..1600, skewed small), padded /
odd row pitches, every fp64 mode, fp32 (both A stagings), accumulate in k-panels, host-buffer
entries (pageable and pinned) and graph replay; uniform, integer and normal
inputs.  EXACT and integer inputs must be bitwise matmul_seq; tensor modes
<= 1e-12 normwise (OZAKI <= 1e-13 on sampled rows), fp32 <= 1e-5.  Prints one
JSON summary; any failure is listed with its case.

    python tools/fuzz_parity.py [seconds] [seed]
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import numpy as np
import torch

import oracle as O
import paper_1012_2273_b200 as P

budget = float(sys.argv[1]) if len(sys.argv) > 1 else 240.0
seed = int(sys.argv[2]) if len(sys.argv) > 2 else 2026
rng = np.random.default_rng(seed)
ctx = P.Context(0)
MODES = {"auto": P.MODE_AUTO, "dmma": P.MODE_DMMA, "dmma_small": P.MODE_DMMA_SMALL,
         "exact": P.MODE_EXACT, "ozaki": P.MODE_OZAKI}


def bits(x):
    return np.ascontiguousarray(x).view(np.uint64 if x.dtype == np.float64 else np.uint32)


def normwise(x, y):
    d = np.linalg.norm(y)
    return float(np.linalg.norm(x - y) / d) if d else float(np.linalg.norm(x))


def dim():
    r = rng.random()
    if r < 0.01:  # big enough for the streamed host path (>= 2 x 148 tiles of 128 x 128)
        return int(rng.integers(2200, 3000))
    if r < 0.35:
        return int(rng.integers(1, 65))
    if r < 0.8:
        return int(rng.integers(65, 513))
    return int(rng.integers(513, 1601))


def padded(a, pad, dtype):
    m, k = a.shape
    full = torch.zeros((m, k + pad), dtype=dtype, device="cuda")
    v = full[:, :k]
    v.copy_(torch.from_numpy(a))
    return v


counts = {}
fails = []
t_end = time.time() + budget
case = 0
while time.time() < t_end:
    case += 1
    m, k, n = dim(), dim(), dim()
    pa, pb = (int(v) if rng.random() < 0.4 else 0 for v in rng.integers(1, 6, size=2))
    dist = [O.DIST_UNIFORM, O.DIST_INT8, O.DIST_NORMAL][int(rng.integers(0, 3))]
    if dist == O.DIST_NORMAL:  # the oracle's normal stream is fp32 (configs[4]): widened
        a = O.fill(dist, 10 * case + 1, m, k, dtype=np.float32).astype(np.float64)
        b = O.fill(dist, 10 * case + 2, k, n, dtype=np.float32).astype(np.float64)
    else:
        a = O.fill(dist, 10 * case + 1, m, k)
        b = O.fill(dist, 10 * case + 2, k, n)
    small = m * n * k <= 3_000_000
    rows = list(range(m)) if small else sorted({0, int(rng.integers(0, m)), m // 2, m - 1})
    want = O.matmul_seq(a, b) if small else O.matmul_rows(rows, a, b)
    exact_ref = dist == O.DIST_INT8  # every summation order is exact

    def check(name, got, bitwise, tol):
        counts[name] = counts.get(name, 0) + 1
        g = got if small else got[rows]
        ok = (bits(g) == bits(want)).all() if bitwise else normwise(g, want) <= tol
        if not ok:
            fails.append({"case": case, "what": name, "shape": [m, k, n], "pads": [pa, pb],
                          "dist": dist, "err": normwise(g, want)})

    A, B = padded(a, pa, torch.float64), padded(b, pb, torch.float64)
    for name, mode in MODES.items():
        if name == "ozaki" and rng.random() < 0.5:
            continue
        got = ctx.dgemm(A, B, mode=mode).cpu().numpy()
        check(f"dgemm_{name}", got, name == "exact" or exact_ref,
              1e-13 if name == "ozaki" else 1e-12)
    # accumulate: K cut at a multiple of 16, the second launch continues C
    if k > 32 and rng.random() < 0.5:
        cut = int(rng.integers(1, k // 16)) * 16
        mode = [P.MODE_AUTO, P.MODE_EXACT, P.MODE_DMMA][int(rng.integers(0, 3))]
        C = ctx.dgemm(A[:, :cut], B[:cut], mode=mode)
        ctx.dgemm(A[:, cut:], B[cut:], C, mode=mode, accumulate=C)
        one = ctx.dgemm(A, B, mode=mode)
        # the documented contract (include/mmws_gpu.h, mmws_gpu_dgemm_acc): in
        # AUTO a piece under the DFMA latency kernel's limit (n, k <= 96) may
        # take another kernel family than the whole
        small = lambda kk: n <= 96 and kk <= 96  # noqa: E731
        same_family = mode != P.MODE_AUTO or small(cut) == small(k) == small(k - cut)
        counts["accumulate_vs_one_call"] = counts.get("accumulate_vs_one_call", 0) + 1
        if same_family and not torch.equal(C.view(torch.int64), one.view(torch.int64)):
            fails.append({"case": case, "what": "accumulate", "shape": [m, k, n], "cut": cut,
                          "mode": mode})
    # host entries (matmul_host and the 1-rank master_run_host), fp64 and fp32
    if rng.random() < 0.3:
        mode = [P.MODE_AUTO, P.MODE_EXACT, P.MODE_DMMA][int(rng.integers(0, 3))]
        f32 = rng.random() < 0.25
        x0, y0 = (a.astype(np.float32), b.astype(np.float32)) if f32 else (a, b)
        xd, yd = torch.from_numpy(x0).cuda(), torch.from_numpy(y0).cuda()
        dev_c = (ctx.sgemm(xd, yd) if f32 else ctx.dgemm(xd, yd, mode=mode)).cpu().numpy()
        for pinned in (False, True):
            x, y = x0, y0
            if pinned:
                x = torch.from_numpy(x0).pin_memory().numpy()
                y = torch.from_numpy(y0).pin_memory().numpy()
            entry = "master_run_host" if rng.random() < 0.3 else "matmul_host"
            c, _ = getattr(ctx, entry)(x, y, mode=P.MODE_FFMA if f32 else mode)
            counts["host_entry_vs_device"] = counts.get("host_entry_vs_device", 0) + 1
            if not (bits(c) == bits(dev_c)).all():
                fails.append({"case": case, "what": entry, "pinned": pinned, "f32": f32,
                              "shape": [m, k, n], "mode": mode})
    # graph replay
    if rng.random() < 0.2:
        C = torch.empty((m, n), dtype=torch.float64, device="cuda")
        g = ctx.graph_dgemm(A, B, C)
        g.launch()
        torch.cuda.synchronize()
        eager = ctx.dgemm(A, B).cpu().numpy()
        counts["graph_vs_eager"] = counts.get("graph_vs_eager", 0) + 1
        if not (bits(C.cpu().numpy()) == bits(eager)).all():
            fails.append({"case": case, "what": "graph", "shape": [m, k, n]})
        g.close()
    # fp32
    af, bf = a.astype(np.float32), b.astype(np.float32)
    Af, Bf = padded(af, pa, torch.float32), padded(bf, pb, torch.float32)
    # A staged as it lies / transposed and staged k-major (default: by size):
    # the same bits either way
    ctx.tune("MMWS_GPU_SGEMM_AT", "1")
    got_at = ctx.sgemm(Af, Bf)
    ctx.tune("MMWS_GPU_SGEMM_AT", "0")
    got_rm = ctx.sgemm(Af, Bf)
    ctx.tune("MMWS_GPU_SGEMM_AT", None)
    counts["sgemm_k_major_bitwise"] = counts.get("sgemm_k_major_bitwise", 0) + 1
    if not bool(torch.equal(got_at.view(torch.int32), got_rm.view(torch.int32))):
        fails.append({"case": case, "what": "sgemm k-major vs row-major", "shape": [m, k, n],
                      "pads": [pa, pb]})
    gotf = (got_at if case % 2 else ctx.sgemm(Af, Bf)).cpu().numpy().astype(np.float64)
    wantf = O.matmul_rows(rows, af, bf)
    counts["sgemm"] = counts.get("sgemm", 0) + 1
    g = gotf[rows]
    ok = (g == wantf).all() if exact_ref else normwise(g, wantf) <= 1e-5
    if not ok:
        fails.append({"case": case, "what": "sgemm", "shape": [m, k, n], "pads": [pa, pb],
                      "err": normwise(g, wantf)})

print(json.dumps({"seed": seed, "seconds": budget, "cases": case, "checks": counts,
                  "checks_total": sum(counts.values()), "failures": fails[:50],
                  "failure_count": len(fails)}))
sys.exit(1 if fails else 0)
