"""Which cuMulticastCreate properties does this box accept?  (ctypes on libcuda)"""
import ctypes

cu = ctypes.CDLL("libcuda.so.1")
assert cu.cuInit(0) == 0
dev = ctypes.c_int()
cu.cuDeviceGet(ctypes.byref(dev), 0)
ctx = ctypes.c_void_p()
cu.cuDevicePrimaryCtxRetain(ctypes.byref(ctx), dev)
cu.cuCtxSetCurrent(ctx)
v = ctypes.c_int()
for attr, name in [(132, "MULTICAST_SUPPORTED"), (129, "HANDLE_TYPE_FABRIC_SUPPORTED?"), (102, "VMM")]:
    r = cu.cuDeviceGetAttribute(ctypes.byref(v), attr, dev)
    print(name, r, v.value)


class Prop(ctypes.Structure):
    _fields_ = [("numDevices", ctypes.c_uint), ("size", ctypes.c_size_t), ("handleTypes", ctypes.c_ulonglong),
                ("flags", ctypes.c_ulonglong)]


for nd in (1, 2):
    for ht in (0, 1, 8, 9):
        for size in (2 << 20, 64 << 20, 512 << 20):
            p = Prop(nd, size, ht, 0)
            g = ctypes.c_size_t()
            rg = cu.cuMulticastGetGranularity(ctypes.byref(g), ctypes.byref(p), 1)
            h = ctypes.c_ulonglong()
            r = cu.cuMulticastCreate(ctypes.byref(h), ctypes.byref(p))
            print(f"numDevices={nd} handleTypes={ht} size={size >> 20}MB gran(rc={rg})={g.value >> 20}MB create rc={r}")
            if r == 0:
                ra = cu.cuMulticastAddDevice(h, dev)
                print("   addDevice rc", ra)
                cu.cuMemRelease(h)
