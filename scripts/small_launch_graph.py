"""Device-only time of single-tensor Adam steps vs size (GPU): 100 launches (step counts 1..100)
captured in one CUDA graph and replayed, so host cost drops out.  Run once per kernel variant
(MPO_LIB_OVERRIDE / MPO_STEP_KERNEL) to compare kernels for small problems.
usage: python scripts/small_launch_graph.py [label]"""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2309_12381_b200 as mpo

label = sys.argv[1] if len(sys.argv) > 1 else "default"
out = {"label": label}
K = 100
for lg in (14, 16, 18, 20, 21, 22, 23, 24, 26):
    n = 1 << lg
    v = (torch.randn(n, device="cuda") * 0.02).to(torch.float16)
    r = torch.zeros(n, dtype=torch.int16, device="cuda")
    g = (torch.randn(n, device="cuda") * 1e-3).to(torch.float16)
    m, vv = torch.zeros(n, device="cuda"), torch.zeros(n, device="cuda")
    tab = mpo.TensorTable([v], [r], [g], [m], [vv])
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        mpo.mpo_adam_step(tab, mpo.AdamParams(lr=1e-3, step=1))
        torch.cuda.synchronize()
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph, stream=s):
            for t in range(1, K + 1):
                mpo.mpo_adam_step(tab, mpo.AdamParams(lr=1e-3, step=t))
    graph.replay()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 5
    a.record()
    for _ in range(reps):
        graph.replay()
    b.record()
    torch.cuda.synchronize()
    us = a.elapsed_time(b) / (reps * K) * 1e3
    out[f"2^{lg}"] = {"us": round(us, 2), "gbs": round(26 * n / (us * 1e-6) / 1e9)}
    del graph, tab, v, r, g, m, vv
    torch.cuda.empty_cache()
print(json.dumps(out))
