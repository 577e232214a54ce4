"""`index build` of the reference's command-line tool (p/tools/ndcli.cpp:137-180)
on the B200 path:

  python -m paper_1709_07781_b200.cli index build --rows 3000 --cardinality 7 \\
      --seed 5 --verify --output idx.wah [--input values.raw|values.txt] [--runs N]

Values come from --input (raw little-endian u32, or text one value per line,
wah_index_io.cpp:89-105) or from the reference's generator (mt19937(seed),
uniform over [0, cardinality)).  The build runs through the compute-actor
chain (libndactor.so).  --verify decodes every value's bitmap back on the GPU
and checks that the bitmaps reproduce the column exactly (each row set in
exactly its own value's bitmap); --output writes the "WAH1" file
(wah_index_io.cpp:30-44).
"""
from __future__ import annotations

import argparse
import os
import sys
import time

import numpy as np


def read_values(path: str) -> np.ndarray:
    if path.endswith(".txt"):
        with open(path) as f:
            return np.array([int(x) for x in f.read().split()], dtype=np.uint32)
    return np.fromfile(path, dtype="<u4").astype(np.uint32)


def verify(row_count: int, entries: np.ndarray, words: np.ndarray, values: np.ndarray) -> None:
    """GPU round trip: every value's decoded rows are exactly its rows."""
    import torch

    from . import query

    d_words = torch.from_numpy(np.ascontiguousarray(words, np.uint32).view(np.int32).copy()).cuda()
    idx = query.DeviceIndex(row_count, entries, d_words)
    seen = np.zeros(row_count, np.uint8)
    for v, off, ln in entries.tolist():
        rows = idx.rows_for(v)
        if rows.size == 0 or not np.all(values[rows] == v):
            raise SystemExit(f"verify: value {v} decodes to rows holding other values")
        seen[rows] += 1
    if not np.all(seen == 1):
        raise SystemExit("verify: the bitmaps do not partition the rows")


def index_build(a) -> int:
    from . import gen
    from .runtime import Runtime

    values = read_values(a.input) if a.input else gen.uniform(a.seed, a.rows, max(a.cardinality, 1))
    rt = Runtime()
    entries = words = None
    for run in range(a.runs):
        t0 = time.perf_counter()
        n, entries, words = rt.build_index(values)
        print(f"index rows={values.size} run={run}: {time.perf_counter() - t0:.6f} s")
    bpr = 32.0 * words.size / values.size if values.size else 0.0
    print(f"rows={values.size} distinct={len(entries)} words={words.size} ({bpr:.2f} bits per row)")
    if a.verify:
        verify(values.size, entries, words, values)
        print("verified: every value's bitmap decodes back to its rows (GPU)")
    if a.output:
        rc = rt.lib.ndactor_write_index_file(os.fsencode(a.output), values.size,
                                             entries.ctypes.data if entries.size else None, len(entries),
                                             words.ctypes.data if words.size else None, words.size)
        if rc:
            raise SystemExit("cannot write " + a.output + ": " + rt.lib.ndactor_last_error().decode())
        print(f"wrote index to {a.output}")
    rt.close()
    return 0


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="ndcli")
    ap.add_argument("--seed", type=int, default=1)
    sub = ap.add_subparsers(dest="cmd", required=True)
    ix = sub.add_parser("index").add_subparsers(dest="sub", required=True)
    b = ix.add_parser("build")
    b.add_argument("--rows", type=int, default=1 << 20)
    b.add_argument("--cardinality", type=int, default=256)
    b.add_argument("--input", default="")
    b.add_argument("--output", default="")
    b.add_argument("--verify", action="store_true")
    b.add_argument("--runs", type=int, default=1)
    b.add_argument("--seed", type=int, default=None, dest="seed_sub")
    a = ap.parse_args(argv)
    if a.seed_sub is not None:  # `index build --seed S` or the global `--seed S index build`
        a.seed = a.seed_sub
    return index_build(a)


if __name__ == "__main__":
    sys.exit(main())
