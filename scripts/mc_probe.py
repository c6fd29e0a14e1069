"""Probe (GPU): can this box build a multicast (NVLS) object at world 1?  Device attribute, the
library's single-device multicast allocator, and torch symmetric memory's multicast pointer."""
import ctypes, os, socket, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
torch.cuda.init()
cu = ctypes.CDLL("libcuda.so.1")
v, dev = ctypes.c_int(), ctypes.c_int()
cu.cuDeviceGet(ctypes.byref(dev), 0)
print("CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED:", cu.cuDeviceGetAttribute(ctypes.byref(v), 132, dev), v.value)
from paper_2309_12381_b200 import api
try:
    b = api.NvlsLocalBuffer(1 << 21)
    print("mpo_nvls_alloc_local: ok", hex(b.uc), hex(b.mc))
    b.free()
except Exception as ex:
    print("mpo_nvls_alloc_local:", ex)
import torch.distributed as dist
s = socket.socket(); s.bind(("127.0.0.1", 0)); port = s.getsockname()[1]; s.close()
os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda:0"))
try:
    import torch.distributed._symmetric_memory as symm
    t = symm.empty(1 << 20, dtype=torch.bfloat16, device="cuda")
    h = symm.rendezvous(t, dist.group.WORLD.group_name)
    print("symm multicast_ptr:", hex(int(getattr(h, "multicast_ptr", 0) or 0)))
except Exception as ex:
    print("symm:", type(ex).__name__, ex)
dist.destroy_process_group()
