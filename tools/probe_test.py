import sys, time
sys.path.insert(0, ".")
import numpy as np, torch
from paper_1709_07781_b200.runtime import Runtime
from paper_1709_07781_b200 import gen
rt = Runtime()
def pr(tag):
    rt.dispatch_probe_ex(1000)
    out = []
    for i in range(3):
        r = rt.dispatch_probe_ex(10000); out.append(round(r["actor_ms"] / r["raw_ms"] - 1, 3))
    print(tag, out, flush=True)
pr("fresh")
n = 1 << 28
keys = torch.from_numpy(gen.zipf(42, n, 65536, 1.0).view(np.int32)).cuda()
for i in range(3):
    rt.build_index_device(keys.data_ptr(), n)
rt.synchronize()
pr("after builds")
hk = torch.empty(n, dtype=torch.int32, pin_memory=True).numpy().view(np.uint32)
hw = torch.empty(2 * n, dtype=torch.int32, pin_memory=True).numpy().view(np.uint32)
he = torch.empty(3 * 65536 * 4, dtype=torch.int32, pin_memory=True).numpy().view(np.uint32)
hc = torch.zeros(3, dtype=torch.int64, pin_memory=True).numpy().view(np.uint64)
rt.wait(rt.build_index_async(hk, hw, he, hc))
pr("after async")
