"""Cycle split of the sort's tile phases (experiment build with
-DNDX_SORT_PROF=1).  Usage:
    python tools/variants.py prof=-DNDX_SORT_PROF=1
    NDX_LIB=libndx_prof.so python tools/sort_prof.py C4
Prints, per tile and CTA, the mean cycles of: load, rank, counts+scan,
staging, look-back, scatter (thread 0's clock between the block barriers)."""
import ctypes
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1709_07781_b200 import gen, ndx  # noqa: E402


def main():
    cfg = sys.argv[1] if len(sys.argv) > 1 else "C4"
    v = gen.config_values(cfg, None)
    n = v.size
    b = ndx.WahBuilder(n)
    keys = torch.from_numpy(v.view(np.int32)).cuda()
    calls = b.stage_calls(keys, n)
    fn = b.lib.ndx_sort_prof_read
    fn.argtypes = [ctypes.c_void_p, ctypes.c_int]
    buf = (ctypes.c_ulonglong * 8)()
    for rep in range(4):
        for _, c in calls:
            c()
        torch.cuda.synchronize()
        if rep == 0:
            fn(buf, 1)
    fn(buf, 0)
    tiles = buf[7]
    names = ["load", "rank", "counts+scan", "stage", "lookback", "scatter"]
    tot = sum(buf[i] for i in range(6))
    print(f"{cfg}: {tiles} tiles over 3 builds")
    for i, nm in enumerate(names):
        print(f"  {nm:15s} {buf[i] / tiles:9.0f} cycles/tile  {100 * buf[i] / tot:5.1f}%")
    print(f"  total           {tot / tiles:9.0f} cycles/tile")


if __name__ == "__main__":
    main()
