"""A/B correctness (GPU): a kernel variant must produce the same bits as the default build.
Runs 3 steps of several workloads (ragged tables, SGD-m / Adam / clip, every storage format) in a
subprocess per library and compares SHA-256 digests of value / residual / m / v.
usage: python scripts/ab_equal.py path/to/variant.so"""
import os, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = r'''
import sys, hashlib
sys.path.insert(0, %r)
import torch, bench
h = hashlib.sha256()
for name in ("resnet50_sgd", "gpt2_adamw", "vit_l16_adam_clip", "flat1m_adam"):
    for scheme in (("rne", "rtz", "x8") if name == "gpt2_adamw" else ("rne",)):
        wl = bench.Workload(name, scheme=scheme)
        for _ in range(3):
            wl.step()
        torch.cuda.synchronize()
        for t in (wl.value, wl.resid, wl.m, wl.v):
            if t is not None:
                h.update(t.view(torch.uint8).cpu().numpy().tobytes())
        print(name, scheme, h.hexdigest()[:16], flush=True)
        del wl; torch.cuda.empty_cache()
''' % ROOT
digests = []
for path in ("default", sys.argv[1]):
    env = dict(os.environ)
    if path != "default":
        env["MPO_LIB_OVERRIDE"] = path
    r = subprocess.run([sys.executable, "-c", CHILD], env=env, capture_output=True, text=True)
    print(path, r.stdout.strip().replace("\n", " | "), r.stderr[-300:] if r.returncode else "", flush=True)
    digests.append(r.stdout.strip())
print("EQUAL" if digests[0] == digests[1] and digests[0] else "DIFFERENT")
