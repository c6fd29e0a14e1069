"""Diagnostic (GPU): host-side cost per step vs device time for the ResNet-50 SGD workload."""
import sys, os, time, json
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import bench
import paper_2309_12381_b200 as mpo
from paper_2309_12381_b200 import _lib

wl = bench.Workload("resnet50_sgd")
for _ in range(5):
    wl.step()
torch.cuda.synchronize()
K = 2000
# (a) host loop wall time and device time, no per-step events
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
t0 = time.perf_counter(); s.record()
for _ in range(K):
    wl.step()
e.record(); t1 = time.perf_counter(); torch.cuda.synchronize()
print("python loop: host us/step %.1f  device us/step %.1f" % ((t1 - t0) / K * 1e6, s.elapsed_time(e) / K * 1e3))
# (b) raw ctypes call with prebuilt hp array
L = _lib.load(False)
hp = mpo.SgdParams(lr=0.3, momentum=0.9, weight_decay=2e-4)
arr, nhp = mpo.api._hp_array(hp, _lib.SgdHP)
st = torch.cuda.current_stream().cuda_stream
tab = wl.table
t0 = time.perf_counter(); s.record()
for _ in range(K):
    L.mpo_sgd_step(tab.vdt, tab.gdt, tab.arr, tab.nt, arr, nhp, st)
e.record(); t1 = time.perf_counter(); torch.cuda.synchronize()
print("raw ctypes: host us/step %.1f  device us/step %.1f" % ((t1 - t0) / K * 1e6, s.elapsed_time(e) / K * 1e3))
# (c) CUDA graph of 20 steps
g = torch.cuda.CUDAGraph()
cs = torch.cuda.Stream()
cs.wait_stream(torch.cuda.current_stream())
with torch.cuda.stream(cs):
    with torch.cuda.graph(g, stream=cs):
        for _ in range(20):
            L.mpo_sgd_step(tab.vdt, tab.gdt, tab.arr, tab.nt, arr, nhp, cs.cuda_stream)
torch.cuda.synchronize()
s.record()
for _ in range(K // 20):
    g.replay()
e.record(); torch.cuda.synchronize()
print("graph: device us/step %.1f" % (s.elapsed_time(e) / K * 1e3))
# (d) torch copy of the same byte volume (460 MB read+write split as 230 MB copy)
a = torch.empty(115_000_000, dtype=torch.float16, device="cuda"); b = torch.empty_like(a)
for _ in range(3): b.copy_(a)
s.record()
for _ in range(200): b.copy_(a)
e.record(); torch.cuda.synchronize()
ms = s.elapsed_time(e) / 200
print("torch copy 230MB: us %.1f  GB/s %.0f" % (ms * 1e3, 2 * a.numel() * 2 / (ms * 1e-3) / 1e9))
a = torch.empty(1 << 30, dtype=torch.float16, device="cuda"); b = torch.empty_like(a)
for _ in range(3): b.copy_(a)
s.record()
for _ in range(20): b.copy_(a)
e.record(); torch.cuda.synchronize()
ms = s.elapsed_time(e) / 20
print("torch copy 2GB: us %.1f  GB/s %.0f" % (ms * 1e3, 2 * a.numel() * 2 / (ms * 1e-3) / 1e9))
