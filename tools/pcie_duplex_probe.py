"""PCIe H2D / D2H from pinned memory on this box: one direction at a time and
both at once (two streams), for the sizes of the mid-N host multiplies."""
import json
import torch

for mb in (1, 8, 16, 64, 256):
    n = mb << 20
    hi = torch.empty(n, dtype=torch.uint8).pin_memory()
    ho = torch.empty(n, dtype=torch.uint8).pin_memory()
    d1 = torch.empty(n, dtype=torch.uint8, device="cuda")
    d2 = torch.empty(n, dtype=torch.uint8, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()

    def run(h2d, d2h, reps=20):
        best = 1e9
        for _ in range(reps):
            torch.cuda.synchronize()
            e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
            e0.record()
            s1.wait_event(e0); s2.wait_event(e0)
            if h2d:
                with torch.cuda.stream(s1):
                    d1.copy_(hi, non_blocking=True)
            if d2h:
                with torch.cuda.stream(s2):
                    ho.copy_(d2, non_blocking=True)
            torch.cuda.current_stream().wait_stream(s1); torch.cuda.current_stream().wait_stream(s2)
            e1.record(); torch.cuda.synchronize()
            best = min(best, e0.elapsed_time(e1) * 1e-3)
        return best
    th, td, tb = run(True, False), run(False, True), run(True, True)
    print(json.dumps({"MB": mb, "h2d_GBps": n / th / 1e9, "d2h_GBps": n / td / 1e9,
                      "both_each_GBps": n / tb / 1e9, "both_us": tb * 1e6, "h2d_us": th * 1e6}), flush=True)
