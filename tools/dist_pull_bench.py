"""Times the multi-GPU step's device work on ONE GPU: the C4 column built as
G row shards one after the other, then the merge plan from device counts and
each rank's owned-slice pull (from local buffers here; over NVLink on a real
multi-GPU box).  Usage: python tools/dist_pull_bench.py [G] [log2 n]"""
import ctypes
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1709_07781_b200 import gen, ndx, shard  # noqa: E402


def main():
    g = int(sys.argv[1]) if len(sys.argv) > 1 else 8
    n = 1 << (int(sys.argv[2]) if len(sys.argv) > 2 else 28)
    v = gen.zipf(42, n, 65536, 1.0)
    L = ndx.load()
    P = ndx._ptr
    b = shard.shard_bounds(n, g).astype(np.int64)
    sb = shard.ShardBuilder(int(np.max(np.diff(b))))
    cap = 1 << 16
    metas = torch.zeros(g * cap * 8, dtype=torch.int32, device="cuda")
    counts = np.zeros((g, 3), np.uint64)
    staged = []
    for k in range(g):
        part = v[b[k]:b[k + 1]]
        keys = torch.from_numpy(part.view(np.int32).copy()).cuda()
        W, D, meta = sb.build(keys, part.size, int(b[k]))
        metas[k * cap * 8: k * cap * 8 + D * 8] = meta[: D * 8]
        counts[k, 1] = D
        staged.append(sb.words[:W].clone())
    dev = torch.device("cuda")
    d_counts = torch.from_numpy(counts.view(np.int32).copy()).to(dev)
    rec = g * cap
    entries = torch.empty(3 * rec + 3, dtype=torch.int32, device=dev)
    merged = torch.empty((rec + 1) * 6, dtype=torch.int32, device=dev)
    totals = torch.zeros(8, dtype=torch.int32, device=dev)
    bounds = torch.zeros(2 * (g + 1), dtype=torch.int32, device=dev)
    scr = torch.empty(L.ndx_dist_plan_scratch_bytes(g, cap) // 4 + 64, dtype=torch.int32, device=dev)
    out = torch.empty(2 * n, dtype=torch.int32, device=dev)
    s = torch.cuda.current_stream().cuda_stream
    srcs = (ctypes.c_void_p * g)(*[t.data_ptr() for t in staged])
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    for rep in range(4):
        ev[0].record()
        ndx.check(L.ndx_dist_plan(P(metas), cap, P(d_counts), g, P(entries), P(merged), P(totals), P(bounds),
                                  P(scr), s), "plan")
        ev[1].record()
        for h in range(g):
            ndx.check(L.ndx_dist_pull(srcs, g, P(merged), rec, P(totals), P(bounds), h, 0, P(out), 2 * n,
                                      2 * n // g, s), "pull")
        ev[2].record()
        torch.cuda.synchronize()
    tot = totals.cpu().numpy().view(np.uint64)
    W = int(tot[1])
    plan_ms, pull_ms = ev[0].elapsed_time(ev[1]), ev[1].elapsed_time(ev[2])
    print(f"G={g} n={n} W={W} D={int(tot[0])} err={int(tot[2])}: plan {plan_ms * 1e3:.0f} us, "
          f"pull of all {g} slices {pull_ms * 1e3:.0f} us ({8 * W / (pull_ms * 1e-3) / 1e9:.0f} GB/s r+w)")


if __name__ == "__main__":
    main()
