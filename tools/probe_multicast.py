"""NVLS multicast probe: can this box create a multicast object
(cuMulticastCreate) for the fused multimem.st all-gather epilogue of SURVEY 8(f) f2?"""
import ctypes
cu = ctypes.CDLL("libcuda.so.1")
cu.cuInit(0)
dev = ctypes.c_int(); cu.cuDeviceGet(ctypes.byref(dev), 0)
ctx = ctypes.c_void_p(); cu.cuDevicePrimaryCtxRetain(ctypes.byref(ctx), dev); cu.cuCtxSetCurrent(ctx)
class MCProp(ctypes.Structure):
    _fields_ = [("numDevices", ctypes.c_uint), ("size", ctypes.c_size_t), ("handleTypes", ctypes.c_ulonglong),
                ("flags", ctypes.c_ulonglong)]
for nd in (1, 2):
    for ht in (0, 1, 8, 9):
        for sz in (2 << 20, 512 << 20):
            p = MCProp(nd, sz, ht, 0)
            h = ctypes.c_ulonglong()
            r = cu.cuMulticastCreate(ctypes.byref(h), ctypes.byref(p))
            extra = ""
            if r == 0:
                extra = " add=%d" % cu.cuMulticastAddDevice(h, dev)
            s = ctypes.c_char_p()
            cu.cuGetErrorName(r, ctypes.byref(s))
            print(nd, ht, sz, r, s.value, extra)
