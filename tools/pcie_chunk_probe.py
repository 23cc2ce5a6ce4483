"""PCIe H2D from pinned memory: one 16 MB copy vs the same bytes as back-to-back
chunks on one stream (1 MB .. 8 MB), and as 2-D copies of 4 KB rows."""
import json
import torch

n = 16 << 20
hi = torch.empty(n, dtype=torch.uint8).pin_memory()
d = torch.empty(n, dtype=torch.uint8, device="cuda")
s = torch.cuda.Stream()


def timed(fn, reps=20):
    best = 1e9
    for _ in range(reps):
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(s):
            torch.cuda._sleep(200000)
            e0.record(s)
            fn()
            e1.record(s)
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1) * 1e-3)
    return best


for chunk_mb in (16, 8, 4, 2, 1, 0.5, 0.25):
    c = int(chunk_mb * (1 << 20))

    def fn():
        for o in range(0, n, c):
            d[o:o + c].copy_(hi[o:o + c], non_blocking=True)
    t = timed(fn)
    print(json.dumps({"chunk_MB": chunk_mb, "copies": n // c, "us": round(t * 1e6, 1),
                      "GBps": round(n / t / 1e9, 1)}), flush=True)
