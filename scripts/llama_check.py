"""Diagnostic (GPU): LLaMA-7B Adam step, multi-tensor table vs mpo_sharded_step(world 1), and copy peak."""
import sys, os, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch, bench
wl = bench.Workload("llama7b_adam")
for mode in ("table", "sharded", "table"):
    f = (lambda: wl.step()) if mode == "table" else (lambda: wl.step(sharded=True))
    ms, per, n = bench.timed(f, 30, 3)
    print(mode, "ms/step %.3f  GB/s %.0f" % (ms, wl.P * 26 / (ms * 1e-3) / 1e9), flush=True)
del wl; torch.cuda.empty_cache()
a = torch.empty(4 << 30, dtype=torch.float16, device="cuda"); b = torch.empty_like(a)
for _ in range(3): b.copy_(a)
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
for _ in range(10): b.copy_(a)
e.record(); torch.cuda.synchronize()
ms = s.elapsed_time(e) / 10
print("torch copy 8GB: GB/s %.0f" % (2 * a.numel() * 2 / (ms * 1e-3) / 1e9))
