"""Single-tensor Adam step time vs size (GPU), for the small launches of hook mode and config C1:
back to back (L2-resident when small) and rotating through >= 4 x L2 of sets (HBM).  Run once per
library variant (MPO_LIB_OVERRIDE / MPO_STEP_KERNEL) to compare kernels for small problems.
usage: python scripts/small_launch.py [label]"""
import json, math, sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2309_12381_b200 as mpo

label = sys.argv[1] if len(sys.argv) > 1 else "default"
L2 = 126 * 2 ** 20
out = {"label": label}
for lg in (14, 16, 18, 20, 21, 22, 23, 24):
    n = 1 << lg
    per = 26 * n
    sets = max(1, int(math.ceil(4 * L2 / per)) + 1) if per < 4 * L2 else 1
    tabs = []
    for k in range(sets):
        v = (torch.randn(n, device="cuda") * 0.02).to(torch.float16)
        r = torch.zeros(n, dtype=torch.int16, device="cuda")
        g = (torch.randn(n, device="cuda") * 1e-3).to(torch.float16)
        m, vv = torch.zeros(n, device="cuda"), torch.zeros(n, device="cuda")
        tabs.append((mpo.TensorTable([v], [r], [g], [m], [vv]), (v, r, g, m, vv)))
    hp = mpo.AdamParams(lr=1e-3, step=1)
    res = {}
    for mode in ("b2b", "rot"):
        it = [0]
        def fn():
            t = tabs[0][0] if mode == "b2b" else tabs[it[0] % sets][0]
            it[0] += 1
            mpo.mpo_adam_step(t, hp)
        for _ in range(10):
            fn()
        iters = 400 if lg <= 20 else 100
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize(); a.record()
        for _ in range(iters):
            fn()
        b.record(); torch.cuda.synchronize()
        us = a.elapsed_time(b) / iters * 1e3
        res[mode] = {"us": round(us, 2), "gbs": round(per / (us * 1e-6) / 1e9)}
    out[f"2^{lg}"] = res
    del tabs
    torch.cuda.empty_cache()
print(json.dumps(out))
