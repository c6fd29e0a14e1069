"""Diagnostic (GPU): which live CUDA tensors make up the hook-mode GPT-2 persistent memory beyond
value + residual + m + v (bench hook_mode_secondary)."""
import gc, os, sys, collections
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import paper_2309_12381_b200 as mpo
from transformers import GPT2Config, GPT2LMHeadModel
dev = torch.device("cuda")
torch.cuda.synchronize()
base = torch.cuda.memory_allocated()
model = GPT2LMHeadModel(GPT2Config()).to(dev)
P = sum(p.numel() for p in model.parameters())
print("after model fp32", (torch.cuda.memory_allocated() - base) / P)
opt = mpo.ResidualAdamW(model.parameters(), fmt=torch.bfloat16, lr=6e-4, betas=(0.9, 0.95), weight_decay=0.1)
gc.collect(); torch.cuda.synchronize()
print("after optimizer", (torch.cuda.memory_allocated() - base) / P)
opt.install_backward_hooks()
idx = torch.randint(0, 50257, (8, 1024), device=dev)
for _ in range(2):
    with torch.autocast("cuda", dtype=torch.bfloat16):
        out = model(idx, labels=idx)
    out.loss.backward()
    del out
gc.collect(); torch.cuda.synchronize()
print("after 2 hook steps", (torch.cuda.memory_allocated() - base) / P)
known = set()
for p in model.parameters():
    known.add(p.data_ptr())
    st = opt.state[p]
    for k in ("resid", "m", "v"):
        if st.get(k) is not None:
            known.add(st[k].data_ptr())
tot = collections.Counter()
for o in gc.get_objects():
    try:
        if torch.is_tensor(o) and o.is_cuda and o.data_ptr() not in known:
            tot[(tuple(o.shape), str(o.dtype), type(o).__name__)] += o.untyped_storage().nbytes()
    except Exception:
        pass
for k, v in tot.most_common(15):
    print(k, v, round(v / P, 4))
for name, b in model.named_buffers():
    print("buffer", name, tuple(b.shape), b.dtype)
    break
print("buffers total B/param", sum(b.untyped_storage().nbytes() for b in model.buffers()) / P)
print(torch.cuda.memory_summary(abbreviated=True)[:1500])
