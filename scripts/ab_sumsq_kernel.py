import sys, os, json, subprocess
CHILD = r'''
import sys, json
sys.path.insert(0, %r)
import torch, bench
wl = bench.Workload("vit_l16_adam_clip")
ms, n = bench.timed(wl.step, 300, 10)
print(json.dumps({"ms": round(ms, 5), "gbs": round(wl.P * wl.bytes_per_param / (ms * 1e-3) / 1e9)}))
''' % os.getcwd()
for rep in range(3):
    for name, env in (("lsu (default)", {}), ("tma", {"MPO_SUMSQ_KERNEL": "tma"})):
        e = dict(os.environ); e.update(env)
        r = subprocess.run([sys.executable, "-c", CHILD], env=e, capture_output=True, text=True)
        print(rep, name, [l for l in r.stdout.splitlines() if l.startswith("{")][-1:] or r.stderr[-300:], flush=True)
