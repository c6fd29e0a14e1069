"""A/B (GPU): the stochastic-rounding storage variant on the GPT-2 AdamW parameter set (fp16),
alternating library builds in fresh processes.  usage: python scripts/ab_sr.py NAME=path.so ..."""
import json, os, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = r'''
import sys, json
sys.path.insert(0, %r)
import bench
bench.WORKLOADS["gpt2_adamw_fp16"] = ("gpt2_small", "fp16") + bench.WORKLOADS["gpt2_adamw"][2:]
r = bench._secondary_one("gpt2_adamw_fp16", 200, 5, 6539.2, scheme="sr")
print(json.dumps({"gbs": round(r["achieved_gbs_step"]), "frac": round(r["frac_of_measured_hbm"], 3)}))
''' % ROOT
for rep in range(2):
    for name, path in (a.split("=", 1) for a in sys.argv[1:]):
        env = dict(os.environ)
        if path != "default":
            env["MPO_LIB_OVERRIDE"] = path
        r = subprocess.run([sys.executable, "-c", CHILD], env=env, capture_output=True, text=True)
        line = [l for l in r.stdout.splitlines() if l.startswith("{")]
        print(rep, name, line[-1] if line else r.stderr[-800:], flush=True)
