import ctypes
cudart = ctypes.CDLL("libcudart.so.12")
v = ctypes.c_int()
for name, attr in [("MaxPersistingL2CacheSize", 108), ("MaxAccessPolicyWindowSize", 109), ("L2CacheSize", 38)]:
    cudart.cudaDeviceGetAttribute(ctypes.byref(v), attr, 0)
    print(name, v.value)
