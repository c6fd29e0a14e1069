import os, torch, torch.distributed as dist
os.environ.setdefault("MASTER_ADDR", "127.0.0.1"); os.environ.setdefault("MASTER_PORT", "29533")
dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda:0"))
import torch.distributed._symmetric_memory as symm
print("has", [a for a in dir(symm) if not a.startswith("__")][:40])
try:
    t = symm.empty(1 << 20, dtype=torch.bfloat16, device="cuda")
    h = symm.rendezvous(t, dist.group.WORLD)
    print("buffer_ptrs", h.buffer_ptrs, "multicast_ptr", getattr(h, "multicast_ptr", None), "world", h.world_size)
except Exception as e:
    print("symm error", type(e).__name__, e)
try:
    import ctypes
    cu = ctypes.CDLL("libcuda.so.1")
    dev = ctypes.c_int(0); val = ctypes.c_int(-1)
    # CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED = 132
    r = cu.cuDeviceGetAttribute(ctypes.byref(val), 132, dev)
    print("multicast supported attr", r, val.value)
except Exception as e:
    print("cu error", e)
dist.destroy_process_group()
