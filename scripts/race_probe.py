import os, sys
sys.path.insert(0, os.getcwd())
import torch
import paper_2309_12381_b200 as mpo
os.environ["MPO_STEP_KERNEL"] = "tma"
n = 148 * 12 * 4096
v, r = mpo.mpo_split(torch.randn(n, device="cuda") * 0.02, torch.bfloat16)
g = (torch.randn(n, device="cuda") * 1e-2).to(torch.bfloat16)
m, w = torch.zeros(n, device="cuda"), torch.zeros(n, device="cuda")
mpo.mpo_adam_step(mpo.TensorTable([v], [r], [g], [m], [w]), mpo.AdamParams(lr=1e-3, step=1))
torch.cuda.synchronize()
print("ok")
