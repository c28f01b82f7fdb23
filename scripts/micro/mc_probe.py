import ctypes
cu = ctypes.CDLL("libcuda.so.1")
cu.cuInit(0)
dev = ctypes.c_int()
cu.cuDeviceGet(ctypes.byref(dev), 0)
v = ctypes.c_int()
# CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED = 132, CU_DEVICE_ATTRIBUTE_HANDLE_TYPE_FABRIC_SUPPORTED = 128
for name, a in (("MULTICAST_SUPPORTED", 132), ("HANDLE_TYPE_FABRIC_SUPPORTED", 128), ("HANDLE_TYPE_POSIX_FD_SUPPORTED", 102)):
    r = cu.cuDeviceGetAttribute(ctypes.byref(v), a, dev)
    print(name, "rc", r, "value", v.value)
