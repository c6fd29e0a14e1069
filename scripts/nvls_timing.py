"""The NVLS fused sharded step's kernel with its multicast operations EMULATED over peer buffers of
one device (mpo_nvls_emulated_step; its HBM side only -- real multimem traffic needs a multi-GPU
box) vs the P2P fused step and the step kernel on the same shard, 1/2/4/8 emulated ranks, rank 0's
launch timed (200 launches, CUDA events).  Each library variant runs in its own process.
usage: python scripts/nvls_timing.py [NAME=path.so ...]   (default: the current exact build)"""
import json, os, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = r'''
import sys, json
sys.path.insert(0, %r)
import torch
import paper_2309_12381_b200 as mpo
from paper_2309_12381_b200 import api
from paper_2309_12381_b200._lib import MPO_ADAM, MPO_SGD
from synth import workloads
for wl_name, kind, tdt in (("resnet50", "sgd", torch.float16), ("gpt2_small", "adam", torch.bfloat16)):
    P = workloads.total(wl_name)
    for world in (1, 2, 4, 8):
        n = (P + 8 * world - 1) // (8 * world) * 8 * world
        S = n // world
        V = [torch.randn(n, device="cuda").to(tdt) * 0.02 for _ in range(world)]
        G = [torch.randn(n, device="cuda").to(tdt) * 1e-3 for _ in range(world)]
        R = torch.zeros(S, dtype=torch.int16, device="cuda")
        M = torch.zeros(S, device="cuda")
        W = torch.zeros(S, device="cuda") if kind == "adam" else None
        hp = mpo.AdamParams(lr=1e-3, grad_scale=1.0 / world) if kind == "adam" else \
            mpo.SgdParams(lr=0.1, momentum=0.9, grad_scale=1.0 / world)
        vp = [t.data_ptr() for t in V]; gp = [t.data_ptr() for t in G]
        k = MPO_ADAM if kind == "adam" else MPO_SGD
        fns = (("nvls_emulated", lambda: api.mpo_nvls_emulated_step(k, 0, world, vp, gp, R, M, W, n, hp, tdt)),
               ("p2p", lambda: api.mpo_p2p_sharded_step(k, 0, world, vp, gp, R, M, W, n, hp, tdt)))
        for name, fn in fns:
            for _ in range(5): fn()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            iters = 200
            torch.cuda.synchronize(); a.record()
            for _ in range(iters): fn()
            b.record(); torch.cuda.synchronize()
            us = a.elapsed_time(b) / iters * 1e3
            # HBM bytes of rank 0's launch: its shard's local streams + every rank's grad slice read
            # + every replica's value slice written
            local = {"adam": 2 + 2 + 8 + 8, "sgd": 2 + 2 + 4 + 4}[kind]
            nb = S * (local + 2 * world + 2 * world)
            print(json.dumps({"variant": %r, "fn": name, "workload": wl_name, "kind": kind, "world": world,
                              "shard": S, "us": round(us, 2), "hbm_gbs": round(nb / us / 1e3, 1)}), flush=True)
        del V, G, R, M, W
        torch.cuda.empty_cache()
''' % (ROOT, 'VARIANT')
variants = [a.split("=", 1) for a in sys.argv[1:]] or [("current", "default")]
for rep in range(2):
    for name, path in variants:
        env = dict(os.environ)
        if path != "default":
            env["MPO_LIB_OVERRIDE"] = path
        r = subprocess.run([sys.executable, "-c", CHILD.replace("'VARIANT'", repr(name))], env=env,
                           capture_output=True, text=True)
        print(r.stdout.strip(), flush=True)
        if r.returncode:
            print(r.stderr[-1500:])
