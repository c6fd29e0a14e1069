"""Diagnostic (GPU): SGD-momentum step time vs size on one flat fp16 tensor (18 B/param), next to
a torch copy moving the same bytes; least-squares t = a + b*bytes gives the per-launch fixed cost
a and the asymptotic bandwidth 1/b of each."""
import json, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import bench
import paper_2309_12381_b200 as mpo
res = {"sgd": [], "copy": []}
for n in (1 << 22, 1 << 23, 25557032, 1 << 25, 1 << 26, 1 << 27, 1 << 28):
    v = torch.randn(n, device="cuda").to(torch.float16)
    r = torch.zeros(n, dtype=torch.int16, device="cuda")
    g = (torch.randn(n, device="cuda") * 1e-2).to(torch.float16)
    m = torch.zeros(n, device="cuda")
    tab = mpo.TensorTable([v], [r], [g], [m], [None])
    hp = mpo.SgdParams(lr=0.3, momentum=0.9, weight_decay=2e-4)
    k = max(20, int(2e9 / (18 * n)))
    ms, _ = bench.timed(lambda: mpo.mpo_sgd_step(tab, hp), k, 10)
    res["sgd"].append((n * 18, ms))
    del v, r, g, m, tab
    a = torch.empty(n * 9 // 2, dtype=torch.float16, device="cuda")
    b = torch.empty_like(a)
    ms, _ = bench.timed(lambda: b.copy_(a), k, 10)
    res["copy"].append((n * 18, ms))
    del a, b
    torch.cuda.empty_cache()
out = {}
for name, pts in res.items():
    xs = [p[0] for p in pts]; ys = [p[1] * 1e-3 for p in pts]
    mx, my = sum(xs) / len(xs), sum(ys) / len(ys)
    bb = sum((x - mx) * (y - my) for x, y in zip(xs, ys)) / sum((x - mx) ** 2 for x in xs)
    aa = my - bb * mx
    out[name] = {"fixed_us": aa * 1e6, "asymptotic_GBps": 1 / bb / 1e9,
                 "points": [{"bytes": x, "us": round(y * 1e6, 2), "GBps": round(x / y / 1e9)} for x, y in zip(xs, ys)]}
print(json.dumps(out))
