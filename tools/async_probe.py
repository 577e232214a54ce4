import sys, time
sys.path.insert(0, ".")
import numpy as np, torch
from paper_1709_07781_b200.runtime import Runtime
from paper_1709_07781_b200 import gen
n = 1 << 28
rt = Runtime()
hk = torch.empty(n, dtype=torch.int32, pin_memory=True).numpy().view(np.uint32)
gen.zipf(42, n, 65536, 1.0, hk)
hw = [torch.empty(2 * n, dtype=torch.int32, pin_memory=True).numpy().view(np.uint32) for _ in range(2)]
he = [torch.empty(3 * 65536 * 4, dtype=torch.int32, pin_memory=True).numpy().view(np.uint32) for _ in range(2)]
hc = [torch.zeros(3, dtype=torch.int64, pin_memory=True).numpy().view(np.uint64) for _ in range(2)]
rt.wait(rt.build_index_async(hk, hw[0], he[0], hc[0]))
rt.wait(rt.build_index_async(hk, hw[1], he[1], hc[1]))  # both slots warm
pend = []
t00 = time.perf_counter()
for i in range(6):
    t0 = time.perf_counter()
    if len(pend) == 2:
        rt.wait(pend.pop(0))
    t1 = time.perf_counter()
    pend.append(rt.build_index_async(hk, hw[i % 2], he[i % 2], hc[i % 2]))
    t2 = time.perf_counter()
    print(f"step {i}: wait {1e3*(t1-t0):.1f} ms, issue {1e3*(t2-t1):.1f} ms", flush=True)
for t in pend:
    t0 = time.perf_counter(); rt.wait(t); print(f"final wait {1e3*(time.perf_counter()-t0):.1f} ms")
print("per step", (time.perf_counter() - t00) / 6 * 1e3, "ms")
