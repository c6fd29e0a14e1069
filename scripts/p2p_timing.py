"""P2P fused sharded step (mpo_p2p_sharded_step) vs the multi-tensor step kernel on the same shard, at
world 1 and with 2/4/8 ranks EMULATED on one device (peer buffers = other buffers of this GPU, so
the "NVLink" traffic is HBM traffic here).  Each variant runs in its own process (MPO_P2P_KERNEL=lsu
selects the round-1 LSU kernel).  Prints one JSON line per (variant, world, workload).
usage: python scripts/p2p_timing.py"""
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
        def p2p():
            api.mpo_p2p_sharded_step(k, 0, world, vp, gp, R, M, W, n, hp, tdt)
        tab = mpo.TensorTable([V[0][:S]], [R], [G[0][:S]], [M], [W])
        def step():
            if kind == "adam": mpo.mpo_adam_step(tab, hp)
            else: mpo.mpo_sgd_step(tab, hp)
        for name, fn in (("p2p", p2p), ("step_kernel_same_shard", step)):
            if name == "step_kernel_same_shard" and world > 1:
                continue
            for _ in range(5): fn()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            iters = 200
            torch.cuda.synchronize(); a.record()
            for _ in range(iters): fn()
            b.record(); torch.cuda.synchronize()
            us = a.elapsed_time(b) / iters * 1e3
            print(json.dumps({"variant": %r, "fn": name, "workload": wl_name, "kind": kind, "world": world,
                              "shard": S, "us": round(us, 2)}), flush=True)
        del V, G, R, M, W, tab
        torch.cuda.empty_cache()
''' % (ROOT, 'VARIANT')
for variant in ("tma", "lsu"):
    env = dict(os.environ)
    if variant == "lsu":
        env["MPO_P2P_KERNEL"] = "lsu"
    r = subprocess.run([sys.executable, "-c", CHILD.replace("'VARIANT'", repr(variant))], env=env, capture_output=True, text=True)
    print(r.stdout.strip())
    if r.returncode:
        print(r.stderr[-1500:])
