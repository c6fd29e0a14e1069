"""Hook-mode timeline (GPU): one GPT-2 small training step (B, T configurable) with the optimizer
fused into backward through the native hooks, recorded with torch.profiler (CUPTI; nsys is not in
this image) and exported as a Chrome trace, plus a summary: kernels on the compute stream, this
library's kernels among them, and the device's idle time between the first and the last kernel of
backward -- i.e. whether the per-parameter steps interleave with the backward kernels without
leaving the GPU idle.  Writes gpurun_out/hook_trace_B{B}_T{T}.json.gz and prints JSON.
usage: python scripts/hook_trace.py [B] [T]"""
import gzip, json, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
from torch.profiler import ProfilerActivity, profile
from transformers import GPT2Config, GPT2LMHeadModel
import paper_2309_12381_b200 as mpo

B = int(sys.argv[1]) if len(sys.argv) > 1 else 8
T = int(sys.argv[2]) if len(sys.argv) > 2 else 1024
dev = torch.device("cuda")
torch.manual_seed(0)
idx = torch.randint(0, 50257, (B, T + 1), device=dev)
out = {}
for mode in ("hook", "two_phase"):
    model = GPT2LMHeadModel(GPT2Config()).to(dev)
    opt = mpo.ResidualAdamW(model.parameters(), lr=6e-4, betas=(0.9, 0.95), weight_decay=0.1, fmt=torch.bfloat16)
    if mode == "hook":
        opt.install_backward_hooks()

    def step():
        logits = model(idx[:, :-1]).logits
        loss = torch.nn.functional.cross_entropy(logits.float().reshape(-1, logits.shape[-1]), idx[:, 1:].reshape(-1))
        loss.backward()
        if mode == "two_phase":
            opt.step()
            for p in model.parameters():
                p.grad = None
    for _ in range(3):
        step()
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
        step()
        torch.cuda.synchronize()
    path = os.path.join(ROOT, "gpurun_out", f"hook_trace_{mode}_B{B}_T{T}.json")
    os.makedirs(os.path.dirname(path), exist_ok=True)
    prof.export_chrome_trace(path)
    with open(path, "rb") as f, gzip.open(path + ".gz", "wb") as g:
        g.write(f.read())
    os.unlink(path)
    ev = json.load(gzip.open(path + ".gz"))
    ev = ev["traceEvents"] if isinstance(ev, dict) else ev
    ks = sorted([e for e in ev if e.get("cat") == "kernel"], key=lambda e: e["ts"])
    mine = [e for e in ks if "mpo::" in e["name"]]
    busy = sum(e["dur"] for e in ks)
    span = (ks[-1]["ts"] + ks[-1]["dur"] - ks[0]["ts"]) if ks else 0.0
    # idle time inside the step: gaps between consecutive kernels (single stream)
    idle, end = 0.0, None
    for e in ks:
        if end is not None and e["ts"] > end:
            idle += e["ts"] - end
        end = max(end or 0.0, e["ts"] + e["dur"])
    out[mode] = {"kernels": len(ks), "library_kernels": len(mine), "library_kernel_us": sum(e["dur"] for e in mine),
                 "kernel_busy_us": busy, "first_to_last_kernel_us": span, "idle_between_kernels_us": idle,
                 "trace": os.path.relpath(path + ".gz", ROOT)}
    del model, opt
    torch.cuda.empty_cache()
print(json.dumps({"B": B, "T": T, **out}))
