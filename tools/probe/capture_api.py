"""Probe: which host runtime calls invalidate a stream capture (global mode, torch.cuda.graph)."""
import ctypes
import torch

rt = ctypes.CDLL("libcudart.so.12")
for name in ("cudaStreamGetId", "cudaStreamIsCapturing", "cudaEventCreateWithFlags"):
    print(name, hasattr(rt, name))


def trial(label, fn):
    s = torch.cuda.Stream()
    x = torch.zeros(16, device="cuda")
    g = torch.cuda.CUDAGraph()
    try:
        with torch.cuda.graph(g, stream=s):
            x += 1
            fn(s)
            x += 1
        print(label, "ok")
    except Exception as e:
        print(label, "FAILED", str(e).splitlines()[0])
    torch.cuda.synchronize()


def get_id(s):
    v = ctypes.c_ulonglong()
    r = rt.cudaStreamGetId(ctypes.c_void_p(s.cuda_stream), ctypes.byref(v))
    print("  cudaStreamGetId ->", r)


def is_cap(s):
    v = ctypes.c_int()
    r = rt.cudaStreamIsCapturing(ctypes.c_void_p(s.cuda_stream), ctypes.byref(v))
    print("  cudaStreamIsCapturing ->", r, v.value)


trial("nothing", lambda s: None)
trial("is_capturing", is_cap)
trial("get_id", get_id)
trial("is_capturing then get_id", lambda s: (is_cap(s), get_id(s)))
