"""Diagnostic (GPU): pinned host<->device copy rates for the e2e leg's byte counts (51 MB per
direction per step): H2D alone, D2H alone, both concurrently on two streams, and split in chunks."""
import json, torch
n = 25557032 + 8 * 161
h_in = torch.empty(n, dtype=torch.float16, pin_memory=True)
h_out = torch.empty(n, dtype=torch.float16, pin_memory=True)
d_in = torch.empty(n, dtype=torch.float16, device="cuda")
d_out = torch.empty(n, dtype=torch.float16, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def t(fn, k=30):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(); [fn() for _ in range(k)]; b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / k
def h2d():
    with torch.cuda.stream(s1): d_in.copy_(h_in, non_blocking=True)
    torch.cuda.current_stream().wait_stream(s1)
def d2h():
    with torch.cuda.stream(s2): h_out.copy_(d_out, non_blocking=True)
    torch.cuda.current_stream().wait_stream(s2)
def both():
    with torch.cuda.stream(s1): d_in.copy_(h_in, non_blocking=True)
    with torch.cuda.stream(s2): h_out.copy_(d_out, non_blocking=True)
    torch.cuda.current_stream().wait_stream(s1); torch.cuda.current_stream().wait_stream(s2)
def chunked(c=4):
    k = n // c
    for i in range(c):
        lo, hi = i * k, (n if i == c - 1 else (i + 1) * k)
        with torch.cuda.stream(s1): d_in[lo:hi].copy_(h_in[lo:hi], non_blocking=True)
        with torch.cuda.stream(s2): h_out[lo:hi].copy_(d_out[lo:hi], non_blocking=True)
    torch.cuda.current_stream().wait_stream(s1); torch.cuda.current_stream().wait_stream(s2)
B = n * 2
r = {}
for name, fn in (("h2d", h2d), ("d2h", d2h), ("both", both), ("chunked4", chunked)):
    ms = t(fn)
    r[name] = {"ms": round(ms, 4), "GBps_per_direction": round(B / (ms * 1e-3) / 1e9, 1)}
print(json.dumps(r))
