"""Probe NVLink SHARP / multicast support on this box (driver API via ctypes).

  python tools/probe_nvls.py

Prints CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED per device and tries to create
a multicast object over all visible devices in one process."""
import ctypes as C
import json

cu = C.CDLL("libcuda.so.1")
CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED = 132
CU_DEVICE_ATTRIBUTE_HANDLE_TYPE_FABRIC_SUPPORTED = 128


def ck(r, what):
    if r != 0:
        s = C.c_char_p()
        cu.cuGetErrorString(r, C.byref(s))
        raise RuntimeError(f"{what}: {r} {s.value}")


ck(cu.cuInit(0), "cuInit")
n = C.c_int()
ck(cu.cuDeviceGetCount(C.byref(n)), "count")
out = {"devices": n.value, "multicast": [], "fabric": []}
for d in range(n.value):
    dev = C.c_int()
    ck(cu.cuDeviceGet(C.byref(dev), d), "get")
    v = C.c_int()
    ck(cu.cuDeviceGetAttribute(C.byref(v), CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, dev), "attr")
    out["multicast"].append(v.value)
    ck(cu.cuDeviceGetAttribute(C.byref(v), CU_DEVICE_ATTRIBUTE_HANDLE_TYPE_FABRIC_SUPPORTED, dev),
       "attr")
    out["fabric"].append(v.value)


class McProp(C.Structure):
    _fields_ = [("numDevices", C.c_uint), ("size", C.c_size_t), ("handleTypes", C.c_ulonglong),
                ("flags", C.c_ulonglong)]


try:
    ctx = C.c_void_p()
    dev0 = C.c_int()
    ck(cu.cuDeviceGet(C.byref(dev0), 0), "get")
    ck(cu.cuDevicePrimaryCtxRetain(C.byref(ctx), dev0), "ctx")
    ck(cu.cuCtxSetCurrent(ctx), "setctx")
    prop = McProp(n.value, 0, 1, 0)  # POSIX FD handles
    gran = C.c_size_t()
    ck(cu.cuMulticastGetGranularity(C.byref(gran), C.byref(prop), 1), "granularity")
    prop.size = gran.value * 4
    h = C.c_ulonglong()
    ck(cu.cuMulticastCreate(C.byref(h), C.byref(prop)), "cuMulticastCreate")
    for d in range(n.value):
        dev = C.c_int()
        ck(cu.cuDeviceGet(C.byref(dev), d), "get")
        ck(cu.cuMulticastAddDevice(h, dev), f"cuMulticastAddDevice({d})")
    out["multicast_create"] = "ok"
    out["granularity"] = gran.value
except Exception as ex:  # report, never fail
    out["multicast_create"] = str(ex)
print(json.dumps(out))
