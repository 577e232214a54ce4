"""ctypes binding of the C++ runtime's C ABI (include/ndactor_c.h).

`Runtime` owns one ActorSystem + Device + the four build-stage compute actors
(libndactor.so).  `build_index` is the public host call (host values in, host
index out, through the actor chain); `build_index_device` runs the chain on
device-resident keys and leaves the index in HBM."""
from __future__ import annotations

import ctypes
import os

import numpy as np

from . import _build

_LIB = None
_vp = ctypes.c_void_p
_u32p = ctypes.POINTER(ctypes.c_uint32)
_u64 = ctypes.c_uint64


class RuntimeError_(RuntimeError):
    pass


def lib_path() -> str:
    return os.path.join(_build.LIB, "libndactor.so")


def load() -> ctypes.CDLL:
    global _LIB
    if _LIB is None:
        if not os.path.exists(lib_path()):
            _build.build_all()
        lib = ctypes.CDLL(lib_path())
        sig = {
            "ndactor_runtime_create": (ctypes.c_int, [ctypes.c_int, ctypes.c_uint, ctypes.POINTER(_vp)]),
            "ndactor_runtime_destroy": (None, [_vp]),
            "ndactor_last_error": (ctypes.c_char_p, []),
            "ndactor_runtime_stream": (_vp, [_vp]),
            "ndactor_runtime_synchronize": (ctypes.c_int, [_vp]),
            "ndactor_wah_build_index": (ctypes.c_int, [_vp, _vp, _u64, ctypes.c_uint32, _vp, _u64, _vp, _u64,
                                                       ctypes.POINTER(_u64), ctypes.POINTER(_u64)]),
            "ndactor_wah_build_index_device": (ctypes.c_int, [_vp, _vp, _u64, ctypes.c_uint32, ctypes.POINTER(_vp),
                                                              ctypes.POINTER(_vp), ctypes.POINTER(_vp)]),
            "ndactor_dispatch_probe": (ctypes.c_int, [_vp, _u64, ctypes.POINTER(ctypes.c_double),
                                                      ctypes.POINTER(ctypes.c_double), ctypes.POINTER(_u64)]),
            "ndactor_dispatch_probe_ex": (ctypes.c_int, [_vp, _u64, ctypes.POINTER(ctypes.c_double)]),
            "ndactor_wah_build_index_async": (ctypes.c_int, [_vp, _vp, _u64, _vp, _u64, _vp, _u64, _vp,
                                                             ctypes.POINTER(_u64)]),
            "ndactor_wah_wait": (ctypes.c_int, [_vp, _u64]),
            "ndactor_shard_bounds": (ctypes.c_int, [_u64, ctypes.c_uint32, _vp]),
            "ndactor_merge_plan": (ctypes.c_int, [ctypes.c_uint32, _vp, _vp, _u64, _vp, _vp, ctypes.POINTER(_u64),
                                                  ctypes.POINTER(_u64)]),
            "ndactor_write_index_file": (ctypes.c_int, [ctypes.c_char_p, ctypes.c_uint32, _vp, _u64, _vp, _u64]),
            "ndactor_index_digest": (_u64, [ctypes.c_uint32, _vp, _u64, _vp, _u64]),
            "ndactor_nccl_unique_id": (ctypes.c_int, [_vp]),
            "ndactor_dist_create": (ctypes.c_int, [_vp, ctypes.c_int, ctypes.c_int, _vp, _u64, ctypes.c_uint32, _u64,
                                                   ctypes.POINTER(_vp)]),
            "ndactor_dist_step": (ctypes.c_int, [_vp, _vp, _u64, _u64, ctypes.c_int]),
            "ndactor_dist_outputs": (ctypes.c_int, [_vp, ctypes.POINTER(_vp), ctypes.POINTER(_vp), ctypes.POINTER(_vp),
                                                    ctypes.POINTER(_vp), ctypes.POINTER(_vp)]),
            "ndactor_dist_destroy": (None, [_vp]),
        }
        for name, (rt, args) in sig.items():
            fn = getattr(lib, name)
            fn.restype = rt
            fn.argtypes = args
        _LIB = lib
    return _LIB


def index_digest(row_count: int, entries: np.ndarray, words: np.ndarray) -> int:
    """FNV-1a-64 of the "WAH1" serialization (SURVEY.md App. C digest), in
    native code: entries are (value, offset, length) u32 triples."""
    e = np.ascontiguousarray(entries, dtype=np.uint32).reshape(-1)
    w = np.ascontiguousarray(words, dtype=np.uint32)
    return int(load().ndactor_index_digest(row_count, e.ctypes.data if e.size else None, e.size // 3,
                                           w.ctypes.data if w.size else None, w.size))


def _check(rc: int, what: str) -> None:
    if rc != 0:
        raise RuntimeError_(f"{what}: {load().ndactor_last_error().decode()}")


class Runtime:
    def __init__(self, device: int = 0, workers: int = 2):
        self.lib = load()
        h = _vp()
        _check(self.lib.ndactor_runtime_create(device, workers, ctypes.byref(h)), "runtime_create")
        self.h = h

    def close(self) -> None:
        if self.h:
            self.lib.ndactor_runtime_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def stream(self) -> int:
        return int(self.lib.ndactor_runtime_stream(self.h) or 0)

    def synchronize(self) -> None:
        _check(self.lib.ndactor_runtime_synchronize(self.h), "synchronize")

    def build_index(self, values: np.ndarray, words_out=None, entries_out=None):
        """wah::build_index: host values in, (row_count, entries (D,3), words) out."""
        v = np.ascontiguousarray(values, dtype=np.uint32)
        n = v.size
        words = words_out if words_out is not None else np.empty(max(2 * n, 1), np.uint32)
        ent = entries_out if entries_out is not None else np.empty(max(3 * n, 1), np.uint32)
        nw, ne = _u64(), _u64()
        _check(self.lib.ndactor_wah_build_index(self.h, v.ctypes.data if n else None, n, 0, words.ctypes.data,
                                                words.size, ent.ctypes.data, ent.size, ctypes.byref(nw),
                                                ctypes.byref(ne)), "build_index")
        return n, ent[: 3 * ne.value].reshape(-1, 3), words[: nw.value]

    def build_index_async(self, values: np.ndarray, words_out: np.ndarray, entries_out: np.ndarray,
                          counts_out: np.ndarray) -> int:
        """Pipelined build (ndactor_wah_build_index_async): the arrays must
        stay untouched until wait(ticket); pinned host memory keeps the
        copies at full PCIe speed.  Output sizes are the capacities (a
        result longer than them is cut, counts_out still holds the true
        sizes).  counts_out: 3 x u64 (words, distinct, min | max << 32)."""
        v = values
        t = _u64()
        _check(self.lib.ndactor_wah_build_index_async(
            self.h, v.ctypes.data, v.size, words_out.ctypes.data, words_out.size, entries_out.ctypes.data,
            entries_out.size, counts_out.ctypes.data, ctypes.byref(t)), "build_index_async")
        return t.value

    def wait(self, ticket: int) -> None:
        _check(self.lib.ndactor_wah_wait(self.h, ticket), "wait")

    def build_index_device(self, d_keys: int, n: int, row_base: int = 0):
        """Enqueue the chain on device keys; returns device pointers
        (counts, words, entries), valid until the next call."""
        w, e, c = _vp(), _vp(), _vp()
        _check(self.lib.ndactor_wah_build_index_device(self.h, d_keys, n, row_base, ctypes.byref(w),
                                                       ctypes.byref(e), ctypes.byref(c)), "build_index_device")
        return c.value, w.value, e.value

    def dispatch_probe_ex(self, iters: int = 10000) -> dict:
        out = (ctypes.c_double * 5)()
        _check(self.lib.ndactor_dispatch_probe_ex(self.h, iters, out), "dispatch_probe_ex")
        return {"raw_ms": out[0], "raw_enqueue_ms": out[1], "actor_ms": out[2], "actor_host_only_ms": out[3],
                "counter": int(out[4])}

    def dispatch_probe(self, iters: int = 10000):
        raw, act, chk = ctypes.c_double(), ctypes.c_double(), _u64()
        _check(self.lib.ndactor_dispatch_probe(self.h, iters, ctypes.byref(raw), ctypes.byref(act),
                                               ctypes.byref(chk)), "dispatch_probe")
        return raw.value, act.value, chk.value


class DistBuild:
    """The multi-GPU build of one rank (include/ndactor/wah_dist.hpp):
    shard chain through the runtime's actors, NCCL all-gather of the shard
    metadata, merge plan and word exchange on the GPU -- one call per step,
    nothing waited for on the host."""

    def __init__(self, rt: Runtime, rank: int, nranks: int, nccl_id: bytes, local_cap: int,
                 meta_cap: int = 1 << 16, slice_cap: int = 0):
        self.rt = rt
        self.lib = rt.lib
        self.rank, self.nranks = rank, nranks
        idb = (ctypes.c_uint8 * 128).from_buffer_copy(nccl_id)
        h = _vp()
        slice_cap = slice_cap or 2 * local_cap * nranks
        self.slice_cap = slice_cap
        _check(self.lib.ndactor_dist_create(rt.h, rank, nranks, ctypes.addressof(idb), local_cap, meta_cap,
                                            slice_cap, ctypes.byref(h)), "dist_create")
        self.h = h

    @staticmethod
    def unique_id() -> bytes:
        lib = load()
        buf = (ctypes.c_uint8 * 128)()
        _check(lib.ndactor_nccl_unique_id(ctypes.addressof(buf)), "nccl_unique_id")
        return bytes(buf)

    def step(self, d_keys: int, n: int, row_base: int, gather_all: bool = False) -> None:
        if row_base < 0 or row_base + n > 1 << 32:
            raise ValueError("row ids row_base .. row_base + n - 1 must fit in u32")
        _check(self.lib.ndactor_dist_step(self.h, d_keys, n, row_base, 1 if gather_all else 0), "dist_step")

    def outputs(self) -> dict:
        t, b, e, sl, lw = _vp(), _vp(), _vp(), _vp(), _vp()
        _check(self.lib.ndactor_dist_outputs(self.h, ctypes.byref(t), ctypes.byref(b), ctypes.byref(e),
                                             ctypes.byref(sl), ctypes.byref(lw)), "dist_outputs")
        return {"totals": t.value, "bounds": b.value, "entries": e.value, "slice": sl.value, "local_words": lw.value}

    def close(self) -> None:
        if self.h:
            self.lib.ndactor_dist_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
