import sys, time, ctypes
sys.path.insert(0, ".")
import numpy as np, torch
from paper_1709_07781_b200 import ndx
lib = ndx.load()
W = 448984672
d = torch.zeros(W, dtype=torch.int32, device="cuda")
h = torch.empty(W, dtype=torch.int32, pin_memory=True)
s = torch.cuda.current_stream().cuda_stream
for i in range(3):
    torch.cuda.synchronize(); t = time.perf_counter()
    ndx.check(lib.ndx_memcpy_d2h_async(h.data_ptr(), d.data_ptr(), W * 4, s)); torch.cuda.synchronize()
    print("ndx d2h pinned(torch)", W * 4 / (time.perf_counter() - t) / 1e9, "GB/s")
p = ctypes.c_void_p()
ndx.check(lib.ndx_host_alloc(ctypes.byref(p), W * 4))
for i in range(2):
    torch.cuda.synchronize(); t = time.perf_counter()
    ndx.check(lib.ndx_memcpy_d2h_async(p, d.data_ptr(), W * 4, s)); torch.cuda.synchronize()
    print("ndx d2h pinned(ndx)", W * 4 / (time.perf_counter() - t) / 1e9, "GB/s")
