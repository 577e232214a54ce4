"""Time the pieces of one sharded step on one GPU (world size 1)."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_1709_07781_b200 import gen, shard  # noqa: E402

os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
os.environ.setdefault("MASTER_PORT", "29544")
torch.cuda.set_device(0)
dist.init_process_group("nccl", rank=0, world_size=1)
n = 1 << 28
v = gen.zipf(42, n, 65536, 1.0)
keys = torch.from_numpy(v.view(np.int32)).cuda()
sb = shard.ShardBuilder(n)
out = None
for it in range(4):
    t = [time.perf_counter()]
    W, D, meta_d = sb.build(keys, n, 0)
    torch.cuda.synchronize(); t.append(time.perf_counter())
    t.append(time.perf_counter())
    padded, sizes = shard.exchange_meta_device(meta_d, D)
    t.append(time.perf_counter())
    entries, pieces, nent, total = shard.plan_merge_device(padded, sizes)
    t.append(time.perf_counter())
    if out is None:
        out = torch.empty(total, dtype=torch.int32, device="cuda")
    shard.assemble_slots([sb.words[:W]], pieces, padded.shape[1] // 8, sizes, total, out=out)
    torch.cuda.synchronize(); t.append(time.perf_counter())
    print("build %.2f - %.2f exchange %.2f plan %.2f assemble %.2f ms" %
          tuple((b - a) * 1e3 for a, b in zip(t, t[1:])))
dist.destroy_process_group()
