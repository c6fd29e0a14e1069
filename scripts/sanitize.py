"""Small runs of every kernel family for compute-sanitizer (memcheck / racecheck / synccheck /
initcheck): split/reconstruct, SGD and Adam steps (with clip, found-inf skip, ragged tails, every
storage format), the hook entry and the sharded entry at world 1, the P2P and the emulated NVLS
fused sharded steps, and the graph-replayed step."""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2309_12381_b200 as mpo  # noqa: E402

torch.manual_seed(0)
dev = "cuda"
sizes = [3, 4097, 9000, 16, 17]
for scheme, dt in (("rne", torch.bfloat16), ("rne", torch.float16), ("rtz", torch.bfloat16), ("sr", torch.float16),
                   ("x8", torch.float16)):
    V, R, G, M, W = [], [], [], [], []
    for n in sizes:
        v, r = mpo.mpo_split(torch.randn(n, device=dev) * 0.02, dt, scheme=scheme, seed=1, sr_stream=0)
        V.append(v); R.append(r); G.append((torch.randn(n, device=dev) * 1e-2).to(dt))
        M.append(torch.zeros(n, device=dev)); W.append(torch.zeros(n, device=dev))
    ws = torch.zeros(mpo.norm_ws_doubles(), dtype=torch.float64, device=dev)
    tab = mpo.TensorTable(V, R, G, M, W, scheme=scheme)
    mpo.mpo_adam_step(tab, mpo.AdamParams(lr=1e-3, max_grad_norm=0.1, step=1, seed=3), norm_ws=ws)
    mpo.mpo_adam_step(tab, mpo.AdamParams(lr=1e-3, clip_value=0.01, skip_nonfinite=True, step=2), norm_ws=ws)
    tab2 = mpo.TensorTable(V, R, G, M, [None] * len(sizes), scheme=scheme)
    mpo.mpo_sgd_step(tab2, mpo.SgdParams(lr=0.1, momentum=0.9, first_step=True, skip_nonfinite=True), norm_ws=ws)
    for v, r in zip(V, R):
        mpo.mpo_reconstruct(v, r, scheme=scheme)
# hook mode
model = torch.nn.Sequential(torch.nn.Linear(32, 40), torch.nn.Linear(40, 8)).cuda()
opt = mpo.ResidualAdamW(model.parameters(), lr=1e-3, fmt=torch.bfloat16, skip_nonfinite=True)
opt.install_backward_hooks()
model(torch.randn(4, 32, device=dev, dtype=torch.bfloat16)).float().sum().backward()
opt.found_inf()
# P2P fused sharded step, 2 ranks emulated on this device (separate grad buffers / replicas)
from paper_2309_12381_b200 import api  # noqa: E402
from paper_2309_12381_b200._lib import MPO_ADAM  # noqa: E402
n, W2 = 2 * 4104, 2
reps = [(torch.randn(n, device=dev) * 0.02).to(torch.bfloat16) for _ in range(W2)]
reps[1].copy_(reps[0])
grads = [(torch.randn(n, device=dev) * 1e-2).to(torch.bfloat16) for _ in range(W2)]
for k in range(W2):
    S = n // W2
    api.mpo_p2p_sharded_step(MPO_ADAM, k, W2, [t.data_ptr() for t in reps], [t.data_ptr() for t in grads],
                             torch.zeros(S, dtype=torch.int16, device=dev), torch.zeros(S, device=dev),
                             torch.zeros(S, device=dev), n, mpo.AdamParams(lr=1e-3, step=1), torch.bfloat16)
# round 2: the P2P step with an int8-residual format (16-element bulk granule + 8-element tail)
# and SGD; a step spanning two gradient dtypes (mpo_grad_sumsq + norm_ready); the Python hooks
from paper_2309_12381_b200._lib import MPO_SGD  # noqa: E402
for k in range(W2):
    S = n // W2
    api.mpo_p2p_sharded_step(MPO_SGD, k, W2, [t.data_ptr() for t in reps], [t.data_ptr() for t in grads],
                             torch.zeros(S, dtype=torch.int8, device=dev), torch.zeros(S, device=dev), None, n,
                             mpo.SgdParams(lr=0.1, momentum=0.9), torch.bfloat16, scheme="x8")
ps = [torch.nn.Parameter(torch.randn(m, device=dev) * 0.02) for m in (4100, 77)]
o2 = mpo.ResidualAdamW(ps, lr=1e-3, fmt=torch.float16, max_grad_norm=0.05)
ps[0].grad = (torch.randn(4100, device=dev) * 1e-2).to(torch.float16)
ps[1].grad_dtype = None
ps[1].grad = torch.randn(77, device=dev) * 1e-2
o2.step()
model2 = torch.nn.Sequential(torch.nn.Linear(32, 40), torch.nn.Linear(40, 8)).cuda()
o3 = mpo.ResidualSGD(model2.parameters(), lr=0.1, momentum=0.9, fmt=torch.float16)
o3.install_backward_hooks(native=False, batch_below=0)
model2(torch.randn(4, 32, device=dev, dtype=torch.float16)).float().sum().backward()
# both step kernels on the same small tables (the library picks the per-thread-load kernel for
# launches of <= 640 tiles; MPO_STEP_KERNEL forces either), and a table above the threshold
for forced in ("tma", "lsu"):
    os.environ["MPO_STEP_KERNEL"] = forced
    V, R, G, M, W = [], [], [], [], []
    for n in sizes:
        v, r = mpo.mpo_split(torch.randn(n, device=dev) * 0.02, torch.bfloat16)
        V.append(v); R.append(r); G.append((torch.randn(n, device=dev) * 1e-2).to(torch.bfloat16))
        M.append(torch.zeros(n, device=dev)); W.append(torch.zeros(n, device=dev))
    mpo.mpo_adam_step(mpo.TensorTable(V, R, G, M, W), mpo.AdamParams(lr=1e-3, step=1))
os.environ.pop("MPO_STEP_KERNEL")
big = 700 * 4096 + 5
v, r = mpo.mpo_split(torch.randn(big, device=dev) * 0.02, torch.float16)
mpo.mpo_sgd_step(mpo.TensorTable([v], [r], [(torch.randn(big, device=dev) * 1e-2).to(torch.float16)],
                                 [torch.zeros(big, device=dev)], [None]), mpo.SgdParams(lr=0.1, momentum=0.9))
mpo.mpo_reconstruct(v, r)
# round 2 (late): the NVLS kernel with its multicast operations emulated over 2 ranks' buffers
# (mpo_nvls_emulated_step), the LSU P2P kernel, and the graph-replayed step (eager prepare + step,
# and one captured step replayed)
n2 = 2 * 4104
for k in range(W2):
    S = n2 // W2
    api.mpo_nvls_emulated_step(MPO_ADAM, k, W2, [t.data_ptr() for t in reps], [t.data_ptr() for t in grads],
                               torch.zeros(S, dtype=torch.int16, device=dev), torch.zeros(S, device=dev),
                               torch.zeros(S, device=dev), n2, mpo.AdamParams(lr=1e-3, step=1), torch.bfloat16)
    api.mpo_nvls_emulated_step(MPO_SGD, k, W2, [t.data_ptr() for t in reps], [t.data_ptr() for t in grads],
                               torch.zeros(S, dtype=torch.int16, device=dev), torch.zeros(S, device=dev), None, n2,
                               mpo.SgdParams(lr=0.1, momentum=0.9), torch.bfloat16)
os.environ["MPO_P2P_KERNEL"] = "lsu"
for k in range(W2):
    S = n2 // W2
    api.mpo_p2p_sharded_step(MPO_ADAM, k, W2, [t.data_ptr() for t in reps], [t.data_ptr() for t in grads],
                             torch.zeros(S, dtype=torch.int16, device=dev), torch.zeros(S, device=dev),
                             torch.zeros(S, device=dev), n2, mpo.AdamParams(lr=1e-3, step=1), torch.bfloat16)
os.environ.pop("MPO_P2P_KERNEL")
model3 = torch.nn.Sequential(torch.nn.Linear(32, 40), torch.nn.Linear(40, 8)).cuda().to(torch.bfloat16)
o4 = mpo.ResidualAdamW(model3.parameters(), lr=1e-3, fmt=torch.bfloat16)
o4.enable_graph_step()
xg = torch.randn(4, 32, device=dev, dtype=torch.bfloat16)
model3(xg).float().sum().backward()
o4.prepare_step()
o4.step()
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g):
    o4.step()                                   # captured, nothing executed
for _ in range(2):
    o4.prepare_step()
    g.replay()
torch.cuda.synchronize()
print("sanitize run ok")
