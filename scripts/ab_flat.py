"""A/B (GPU): the ResNet-50 SGD-m step over its 161-tensor table vs the same flat buffers as ONE
tensor (same bytes), per library build, alternating in fresh processes.
usage: python scripts/ab_flat.py NAME=path.so ..."""
import os, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = r'''
import sys, json
sys.path.insert(0, %r)
import torch, bench
import paper_2309_12381_b200 as mpo
wl = bench.Workload("resnet50_sgd")
flat = mpo.TensorTable([wl.value], [wl.resid], [wl.grad], [wl.m], [None])
hp = mpo.SgdParams(**wl.hpkw)
out = {}
for name, fn in (("table161", wl.step), ("flat1", lambda: mpo.mpo_sgd_step(flat, hp)),
                 ("table161_again", wl.step)):
    ms, _ = bench.timed(fn, 3000, 20)
    out[name] = round(ms * 1e3, 2)
print(json.dumps(out))
''' % ROOT
for rep in range(2):
    for name, path in (a.split("=", 1) for a in sys.argv[1:]):
        env = dict(os.environ)
        if path != "default":
            env["MPO_LIB_OVERRIDE"] = path
        r = subprocess.run([sys.executable, "-c", CHILD], env=env, capture_output=True, text=True)
        line = [l for l in r.stdout.splitlines() if l.startswith("{")]
        print(rep, name, "us/step", line[-1] if line else r.stderr[-800:], flush=True)
