import sys, time, os
sys.path.insert(0, os.getcwd())
import torch
import paper_2309_12381_b200 as mpo
from paper_2309_12381_b200 import api, _lib
from paper_2309_12381_b200._lib import AdamHP
n = 1 << 20
v = torch.zeros(n, dtype=torch.float16, device="cuda"); r = torch.zeros(n, dtype=torch.int16, device="cuda")
g = torch.zeros(n, dtype=torch.float16, device="cuda"); m = torch.zeros(n, device="cuda"); w = torch.zeros(n, device="cuda")
tab = mpo.TensorTable([v], [r], [g], [m], [w])
hp = mpo.AdamParams(lr=1e-3, step=1)
N = 20000
def t(name, fn):
    for _ in range(200): fn()
    torch.cuda.synchronize()
    a = time.perf_counter()
    for _ in range(N): fn()
    b = time.perf_counter()
    torch.cuda.synchronize()
    print(f"{name:40s} {1e6*(b-a)/N:7.2f} us/call (host)")
t("AdamParams()", lambda: mpo.AdamParams(lr=1e-3, step=1))
t("_hp_array", lambda: api._hp_array(hp, AdamHP))
t("_stream(None)", lambda: api._stream(None))
t("torch.cuda.current_stream()", lambda: torch.cuda.current_stream())
t("_lib_of", lambda: api._lib_of(True))
L = api._lib_of(True)
arr, nhp = api._hp_array(hp, AdamHP)
s = api._stream(None)
t("raw ctypes mpo_adam_step", lambda: L.mpo_adam_step(tab.vdt, tab.gdt, tab.arr, tab.nt, arr, nhp, None, s))
t("api.mpo_adam_step", lambda: mpo.mpo_adam_step(tab, hp))
t("empty kernel torch (x.add_(0) small)", lambda: m[:16].add_(0))
# where the C call's host time goes: early exit (bad dtype), full validation with an empty table,
# and the launch itself; kernel choice forced to each kernel
t("ctypes call, early EDTYPE exit", lambda: L.mpo_adam_step(99, tab.gdt, tab.arr, tab.nt, arr, nhp, None, s))
t("validation + derive, empty table", lambda: L.mpo_adam_step(tab.vdt, tab.gdt, tab.arr, 0, arr, nhp, None, s))
for kc in ("lsu", "tma"):
    os.environ["MPO_STEP_KERNEL"] = kc
    t(f"full call, {kc} kernel", lambda: L.mpo_adam_step(tab.vdt, tab.gdt, tab.arr, tab.nt, arr, nhp, None, s))
os.environ.pop("MPO_STEP_KERNEL")
small = torch.zeros(4096, dtype=torch.float16, device="cuda")
tab2 = mpo.TensorTable([small], [torch.zeros(4096, dtype=torch.int16, device="cuda")], [small.clone()],
                       [torch.zeros(4096, device="cuda")], [torch.zeros(4096, device="cuda")])
t("full call, 4096 elements", lambda: L.mpo_adam_step(tab2.vdt, tab2.gdt, tab2.arr, tab2.nt, arr, nhp, None, s))
with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CPU, torch.profiler.ProfilerActivity.CUDA]) as prof:
    for _ in range(200):
        L.mpo_adam_step(tab2.vdt, tab2.gdt, tab2.arr, tab2.nt, arr, nhp, None, s)
    torch.cuda.synchronize()
print(prof.key_averages().table(sort_by="cpu_time_total", row_limit=8))
t("api._stream(None) (raw C API)", lambda: api._stream(None))
assert api._stream(None) == torch.cuda.current_stream().cuda_stream
side = torch.cuda.Stream()
with torch.cuda.stream(side):
    assert api._stream(None) == side.cuda_stream
print("stream handles agree")
