"""Synthetic columns (BASELINE configs C1-C5), generated natively by
libndactor.so with the reference's own libstdc++ distributions, so inputs are
bit-identical to the reference's generators (p/tools/ndcli.cpp:144-148,
SURVEY.md Appendix C)."""
from __future__ import annotations

import ctypes
import os

import numpy as np

from . import _build

_LIB = None


def _lib():
    global _LIB
    if _LIB is None:
        path = os.path.join(_build.LIB, "libndactor.so")
        if not os.path.exists(path):
            _build.build_all()
        lib = ctypes.CDLL(path)
        lib.ndactor_gen_uniform.argtypes = [ctypes.c_uint32, ctypes.c_uint64, ctypes.c_uint32, ctypes.c_void_p]
        lib.ndactor_gen_zipf.argtypes = [ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint32, ctypes.c_double,
                                         ctypes.c_void_p]
        lib.ndactor_gen_instances.argtypes = [ctypes.c_uint32, ctypes.c_uint32, ctypes.c_void_p, ctypes.c_uint32,
                                              ctypes.c_uint32, ctypes.c_void_p, ctypes.c_void_p]
        _LIB = lib
    return _LIB


def uniform(seed: int, n: int, cardinality: int, out: np.ndarray | None = None) -> np.ndarray:
    """std::mt19937(seed) + uniform_int_distribution<u32>(0, cardinality-1)."""
    a = out if out is not None else np.empty(max(n, 1), np.uint32)
    _lib().ndactor_gen_uniform(seed, n, cardinality, a.ctypes.data)
    return a[:n]


def zipf(seed: int, n: int, k: int = 65536, s: float = 1.0, out: np.ndarray | None = None) -> np.ndarray:
    """mt19937_64(seed), uniform_real(0,1), inverse CDF of Zipf(s) over k ranks."""
    a = out if out is not None else np.empty(max(n, 1), np.uint32)
    _lib().ndactor_gen_zipf(seed, n, k, s, a.ctypes.data)
    return a[:n]


def instances(seed: int, count: int, cards, max_rows: int) -> list[np.ndarray]:
    """The acceptance gate's instance stream (p/tests/acceptance.cpp:56-63)."""
    c = np.ascontiguousarray(cards, dtype=np.uint32)
    sizes = np.zeros(count, np.uint64)
    L = _lib()
    L.ndactor_gen_instances(seed, count, c.ctypes.data, c.size, max_rows, sizes.ctypes.data, None)
    vals = np.empty(int(sizes.sum()) + 1, np.uint32)
    L.ndactor_gen_instances(seed, count, c.ctypes.data, c.size, max_rows, sizes.ctypes.data, vals.ctypes.data)
    out, pos = [], 0
    for s_ in sizes:
        out.append(vals[pos:pos + int(s_)])
        pos += int(s_)
    return out


# The BASELINE.json configs.
CONFIGS = {
    "C1": dict(n=1 << 20, kind="uniform", seed=1, k=256),
    "C3": dict(n=1 << 26, kind="uniform", seed=1, k=1024),
    "C4": dict(n=1 << 28, kind="zipf", seed=42, k=65536, s=1.0),
    "C5": dict(n=1 << 30, kind="uniform", seed=1, k=65536),
}


def config_values(name: str, n: int | None = None, out: np.ndarray | None = None) -> np.ndarray:
    c = CONFIGS[name]
    n = c["n"] if n is None else n
    if c["kind"] == "uniform":
        return uniform(c["seed"], n, c["k"], out)
    return zipf(c["seed"], n, c["k"], c.get("s", 1.0), out)
