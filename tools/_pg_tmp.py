import json, os, sys
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import numpy as np, torch
import paper_1012_2273_b200 as P
ctx = P.Context(0)
for n in (500, 750, 1000, 1250, 2000, 4096):
    a = np.random.rand(n, n); b = np.random.rand(n, n); c = np.empty((n, n))
    ap = torch.from_numpy(a).pin_memory().numpy(); bp = torch.from_numpy(b).pin_memory().numpy()
    cp = torch.empty((n, n), dtype=torch.float64).pin_memory().numpy()
    res = {}
    reps = 25 if n <= 2000 else 8
    for it in range(reps):
        for kind, x, y, z in (("pin", ap, bp, cp), ("page", a, b, c)):
            _, el = ctx.matmul_host(x, y, out=z)
            res.setdefault(kind, []).append(el * 1e6)
    rec = {"n": n}
    for k, v in res.items():
        v.sort(); rec[k] = {"min": round(v[0], 1), "med": round(v[len(v)//2], 1)}
    print(json.dumps(rec), flush=True)
