"""A/B (GPU): time kernel variants of the step on the same box, alternating, each in a subprocess.
usage: python scripts/ab_variants.py NAME=path.so[,VAR[=VALUE]] ...   (path 'default' = lib/libmpo.so)"""
import json, os, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = r'''
import sys, os, json
sys.path.insert(0, %r)
import torch, bench
out = {}
for name, steps in (("resnet50_sgd", 2000), ("gpt2_adamw", 300), ("llama7b_adam", 20)):
    wl = bench.Workload(name)
    ms, n = bench.timed(wl.step, steps, 5)
    out[name] = round(wl.P * wl.bytes_per_param / (ms * 1e-3) / 1e9)
    del wl; torch.cuda.empty_cache()
print(json.dumps(out))
''' % ROOT
variants = [a.split("=", 1) for a in sys.argv[1:]]
for rep in range(2):
    for name, path in variants:
        env = dict(os.environ)
        if "," in path:                      # name=path,VAR[=VALUE]: also set VAR (workload-side knob)
            path, var = path.split(",", 1)
            k, _, val = var.partition("=")
            env[k] = val or "1"
        if path.startswith("lsu"):
            env["MPO_STEP_KERNEL"] = "lsu"
        elif path != "default":
            env["MPO_LIB_OVERRIDE"] = path
        r = subprocess.run([sys.executable, "-c", CHILD], env=env, capture_output=True, text=True)
        line = [l for l in r.stdout.splitlines() if l.startswith("{")]
        print(rep, name, line[-1] if line else r.stderr[-500:], flush=True)
