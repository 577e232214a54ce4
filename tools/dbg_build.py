"""Small debug build of one generated workload (for compute-sanitizer runs)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import oracle  # noqa: E402
from paper_1709_07781_b200 import gen, ndx  # noqa: E402

n, k = int(sys.argv[1]), int(sys.argv[2])
v = gen.uniform(1, n, k) if k > 0 else gen.zipf(42, n, 65536)
b = ndx.WahBuilder(n)
got = b.build(v)
want = oracle.Port().reference_index(v)
ok = np.array_equal(got.words, want.words) and np.array_equal(got.entries, want.entries)
print("n", n, "k", k, "W", got.words.size, want.words.size, "D", len(got.entries), len(want.entries),
      "OK" if ok else "MISMATCH")
