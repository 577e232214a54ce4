"""Check each stage of the device build separately against numpy/oracle."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
from paper_1709_07781_b200 import gen, ndx  # noqa: E402

kind, n, reps = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]) if len(sys.argv) > 3 else 3
v = gen.zipf(42, n, 65536) if kind == "zipf" else gen.uniform(1, n, int(kind))
order = np.argsort(v, kind="stable").astype(np.uint32)
want = oracle.Port().reference_index(v)
b = ndx.WahBuilder(n)
keys = torch.from_numpy(v.view(np.int32)).cuda()
for rep in range(reps):
    calls = b.stage_calls(keys, n)
    calls[0][1]()
    calls[1][1]()
    torch.cuda.synchronize()
    pr = b.pairs[:2 * n].cpu().numpy().view(np.uint32).reshape(n, 2)
    sk, sr = pr[:, 0], pr[:, 1]
    ok_sort = np.array_equal(sr, order) and np.array_equal(sk, v[order])
    bad = np.nonzero(sr != order)[0]
    calls[2][1]()
    calls[3][1]()
    got = b.fetch(n)
    ok_idx = np.array_equal(got.words, want.words) and np.array_equal(got.entries, want.entries)
    print(f"rep {rep}: sort {'OK' if ok_sort else 'BAD'} ({bad.size} bad, first {bad[:3]}) index {'OK' if ok_idx else 'BAD'}",
          flush=True)
