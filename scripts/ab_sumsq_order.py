"""A/B (GPU): clip pre-pass sweep order -- descending vs ascending -- on the ViT-L/16 Adam + clip
step (BASELINE configs[4]), alternating, each in a fresh process.  The descending sweep (the
pre-pass reads last the tiles the step reads first, so they may still be in L2) was a patch to
sumsq_kernel behind the MPO_SUMSQ_FORWARD knob; measured within noise (profiles/r02_ab_sumsq_order.log)
and not kept, so on the current source both arms run the same ascending kernel.
usage: python scripts/ab_sumsq_order.py"""
import json, os, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
CHILD = r'''
import sys, json
sys.path.insert(0, %r)
import torch, bench
out = {}
for name, steps in (("vit_l16_adam_clip", 300), ("gpt2_adamw", 300)):
    wl = bench.Workload(name)
    ms, n = bench.timed(wl.step, steps, 10)
    out[name] = {"ms": round(ms, 5), "gbs": round(wl.P * wl.bytes_per_param / (ms * 1e-3) / 1e9)}
    del wl; torch.cuda.empty_cache()
print(json.dumps(out))
''' % ROOT
from paper_2309_12381_b200 import _build
_build.build()
fwd = _build.build_variant("sumsq_fwd", ["MPO_SUMSQ_FORWARD"], exact=True)
for rep in range(3):
    for name, path in (("descending (default)", None), ("ascending", fwd)):
        env = dict(os.environ)
        if path:
            env["MPO_LIB_OVERRIDE"] = path
        r = subprocess.run([sys.executable, "-c", CHILD], env=env, capture_output=True, text=True)
        line = [l for l in r.stdout.splitlines() if l.startswith("{")]
        print(rep, name, line[-1] if line else r.stderr[-800:], flush=True)
