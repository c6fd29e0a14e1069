import ctypes, torch
torch.cuda.init()
cu = ctypes.CDLL("libcuda.so.1")
v = ctypes.c_int()
dev = ctypes.c_int()
cu.cuDeviceGet(ctypes.byref(dev), 0)
# CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED = 132
r = cu.cuDeviceGetAttribute(ctypes.byref(v), 132, dev)
print("multicast_supported", r, v.value)
print("device_count", torch.cuda.device_count())
