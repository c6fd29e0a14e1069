"""A/B (GPU): split / reconstruct kernel variants (MPO_LIB_OVERRIDE), alternating, each in a fresh
process; GB/s of algorithmic bytes (8 B/param each way) and a digest of the outputs (must match).
usage: python scripts/ab_conv.py NAME=path.so ...   (path 'default' = the built library)"""
import os, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = r'''
import sys, json, hashlib
sys.path.insert(0, %r)
import torch, bench
import paper_2309_12381_b200 as mpo
out = {}
h = hashlib.sha256()
for lg in (24, 28):
    n = 1 << lg
    g = torch.Generator(device="cuda"); g.manual_seed(7)
    w = torch.randn(n, device="cuda", generator=g) * 0.02
    w[:36] = torch.tensor([0.0, -0.0, 1e-45, 3e38, float("inf"), float("nan")] * 6)
    v = torch.empty(n, dtype=torch.bfloat16, device="cuda"); r = torch.empty(n, dtype=torch.int16, device="cuda")
    o = torch.empty(n, device="cuda")
    for name, fn in (("split", lambda: mpo.mpo_split(w, torch.bfloat16, value=v, resid=r)),
                     ("reconstruct", lambda: mpo.mpo_reconstruct(v, r, out=o))):
        ms, _ = bench.timed(fn, 50, 5)
        out[f"{name}_2^{lg}"] = round(8 * n / (ms * 1e-3) / 1e9)
    torch.cuda.synchronize()
    for t in (v, r, o):
        h.update(t.view(torch.uint8).cpu().numpy().tobytes())
out["digest"] = h.hexdigest()[:16]
print(json.dumps(out))
''' % ROOT
variants = [a.split("=", 1) for a in sys.argv[1:]]
for rep in range(2):
    for name, path in variants:
        env = dict(os.environ)
        if path != "default":
            env["MPO_LIB_OVERRIDE"] = path
        r = subprocess.run([sys.executable, "-c", CHILD], env=env, capture_output=True, text=True)
        line = [l for l in r.stdout.splitlines() if l.startswith("{")]
        print(rep, name, line[-1] if line else r.stderr[-500:], flush=True)
