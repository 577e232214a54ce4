"""PCIe rates on the box: DMA H2D / D2H (pinned) vs the copy-out kernel writing
pinned host memory (ndx_wah_copy_out's path), alone and both directions at once."""
import sys, time
sys.path.insert(0, ".")
import numpy as np, torch
from paper_1709_07781_b200 import ndx

n = 1 << 28
dev = torch.device("cuda")
h_in = torch.empty(n, dtype=torch.int32, pin_memory=True)
d_in = torch.empty(n, dtype=torch.int32, device=dev)
W = 448984672
d_w = torch.zeros(W, dtype=torch.int32, device=dev)
h_w = torch.empty(W, dtype=torch.int32, pin_memory=True)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()

def timeit(f, reps=3):
    f(); torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(reps): f()
    torch.cuda.synchronize()
    return (time.perf_counter() - t) / reps

h2d = timeit(lambda: d_in.copy_(h_in, non_blocking=True))
d2h = timeit(lambda: h_w.copy_(d_w, non_blocking=True))
def both():
    with torch.cuda.stream(s1): d_in.copy_(h_in, non_blocking=True)
    with torch.cuda.stream(s2): h_w.copy_(d_w, non_blocking=True)
bd = timeit(both)
print(f"H2D {4*n/h2d/1e9:.1f} GB/s, D2H {4*W/d2h/1e9:.1f} GB/s, both at once {bd*1e3:.1f} ms "
      f"(H2D alone {h2d*1e3:.1f} ms, D2H alone {d2h*1e3:.1f} ms)")
