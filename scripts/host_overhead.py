"""Host-side cost of one optimizer step (GPU box): ResidualAdamW.step() over GPT-2 small's 148
parameters (grads set), timed with perf_counter around the (asynchronous) call -- i.e. the Python
marshalling + validation + launch cost -- and the same for one hook-mode backward's hooks."""
import os, sys, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2309_12381_b200 as mpo
from synth import workloads
sizes = workloads.sizes("gpt2_small")
ps = [torch.nn.Parameter(torch.randn(n, device="cuda") * 0.02) for n in sizes]
opt = mpo.ResidualAdamW(ps, lr=1e-3, fmt=torch.bfloat16)
for p in ps:
    p.grad = torch.zeros(p.shape, dtype=torch.bfloat16, device="cuda")
for _ in range(5):
    opt.step()
torch.cuda.synchronize()
t = []
for _ in range(50):
    t0 = time.perf_counter(); opt.step(); t.append(time.perf_counter() - t0)
torch.cuda.synchronize()
t.sort()
print(json.dumps({"step_host_us_median": 1e6 * t[len(t) // 2], "step_host_us_min": 1e6 * t[0], "params": len(ps)}))
