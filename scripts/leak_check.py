import gc, sys, weakref, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, torch.nn as nn
import paper_2309_12381_b200 as mpo
torch.cuda.synchronize()
base = torch.cuda.memory_allocated()
def run(batch):
    m = nn.Sequential(nn.Linear(512, 512), nn.LayerNorm(512), nn.Linear(512, 512)).cuda()
    opt = mpo.ResidualAdamW(m.parameters(), lr=1e-3, fmt=torch.bfloat16)
    opt.install_backward_hooks(batch_below=batch)
    loss = m(torch.randn(4, 512, device="cuda", dtype=torch.bfloat16)).float().sum()
    loss.backward()
    return weakref.ref(opt), weakref.ref(m)
for batch in (0, 1 << 16):
    wo, wm = run(batch)
    gc.collect()
    torch.cuda.synchronize()
    print("batch", batch, "opt alive", wo() is not None, "model alive", wm() is not None, "leak bytes", torch.cuda.memory_allocated() - base)
    if wo() is not None:
        for r in gc.get_referrers(wo()):
            print("  referrer", type(r), str(r)[:200])
