"""Per-stage device timing of the 4-stage build (CUDA events on the launch
stream), for iteration on the kernels.  Usage:
    python tools/stage_times.py [C3|C4|C1] [--reps 10] [--check]
"""
import argparse
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1709_07781_b200 import gen, ndx  # noqa: E402
from paper_1709_07781_b200.ndx import _ptr, check  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("config", nargs="?", default="C3")
    ap.add_argument("--n", type=int, default=0)
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--check", action="store_true")
    ap.add_argument("--ref", action="store_true", help="also the oracle's digest of the same values (slow)")
    ap.add_argument("--no-flush", action="store_true", help="builds back to back (as bench.py), no L2 flush")
    ap.add_argument("--stages", type=int, default=4, help="run only the first K stages (experiments)")
    a = ap.parse_args()
    if a.config == "U32":  # general keys (the pairs form): uniform over the whole u32 range
        v = np.random.default_rng(7).integers(0, 1 << 32, a.n or (1 << 26), dtype=np.uint64).astype(np.uint32)
    else:
        v = gen.config_values(a.config, a.n or None)
    n = v.size
    b = ndx.WahBuilder(n)
    keys = torch.from_numpy(v.view(np.int32)).cuda()
    s = torch.cuda.current_stream()
    sh = s.cuda_stream
    L = b.lib
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(5)]
    flush = torch.empty(256 << 20, dtype=torch.int32, device="cuda")
    times = []
    calls = b.stage_calls(keys, n)[:a.stages]
    for rep in range(a.reps + 3):
        if not a.no_flush:
            flush.zero_()
        ev[0].record(s)
        for i, (_, call) in enumerate(calls):
            call()
            ev[i + 1].record(s)
        torch.cuda.synchronize()
        if rep >= 3:
            times.append([ev[i].elapsed_time(ev[i + 1]) for i in range(len(calls))] + [0.0] * (4 - len(calls)))
    t = np.median(np.array(times), axis=0)
    W, D = b.counts() if a.stages == 4 else (0, 0)
    tot = t.sum()
    print(f"{a.config} n={n} W={W} D={D}")
    for name, x in zip(["plan", "sort", "emit", "table"], t):
        print(f"  {name:6s} {x * 1e3:9.1f} us")
    balg = 40 * n + 4 * W + 12 * D
    print(f"  total  {tot * 1e3:9.1f} us  -> {n / tot / 1e6:.2f} G values/s, "
          f"{balg / tot / 1e6:.0f} GB/s on the 40N+4W+12D model")
    if a.check:
        sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
        import oracle

        got = b.fetch(n)
        d = oracle.Port().digest_parts(got.row_count, got.entries, got.words)
        print("  digest %016x" % d)
        if a.ref:
            import time as _t
            t0 = _t.perf_counter()
            r = oracle.Port().digest_of(v)
            print("  oracle %016x (%s, %.0f s)" % (r, "match" if r == d else "MISMATCH", _t.perf_counter() - t0))


if __name__ == "__main__":
    main()
