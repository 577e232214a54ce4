"""ctypes binding of the device C ABI (include/ndx.h, lib/libndx.so).

This is the binding a Python caller of the reference-facing boundary would
write (INTEGRATION.md shows it); tests and bench.py drive the CUDA path
through it.  Device memory comes from torch tensors (plumbing only), every
computation is one of our sm_100a kernels.  There is no CPU fallback: if the
library or a GPU is missing, the calls raise.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import numpy as np

from . import _build

_LIB = None
_vp = ctypes.c_void_p
_u64 = ctypes.c_uint64
_u32 = ctypes.c_uint32
_sz = ctypes.c_size_t


class NdxError(RuntimeError):
    pass


# (name, restype, argtypes) for every entry point declared in include/ndx.h
SIGNATURES = [
    ("ndx_error_string", ctypes.c_char_p, [ctypes.c_int]),
    ("ndx_abi_version", ctypes.c_int, []),
    ("ndx_device_count", ctypes.c_int, [ctypes.POINTER(ctypes.c_int)]),
    ("ndx_device_open", ctypes.c_int, [ctypes.c_int]),
    ("ndx_device_bind", ctypes.c_int, [ctypes.c_int]),
    ("ndx_malloc_shared", ctypes.c_int, [ctypes.POINTER(_vp), _sz]),
    ("ndx_free_shared", ctypes.c_int, [_vp]),
    ("ndx_ipc_handle", ctypes.c_int, [_vp, _vp]),
    ("ndx_ipc_open", ctypes.c_int, [_vp, ctypes.POINTER(_vp)]),
    ("ndx_ipc_close", ctypes.c_int, [_vp]),
    ("ndx_device_sm_count", ctypes.c_int, [ctypes.c_int, ctypes.POINTER(ctypes.c_int)]),
    ("ndx_device_synchronize", ctypes.c_int, []),
    ("ndx_stream_create", ctypes.c_int, [ctypes.POINTER(_vp)]),
    ("ndx_stream_destroy", ctypes.c_int, [_vp]),
    ("ndx_stream_synchronize", ctypes.c_int, [_vp]),
    ("ndx_stream_query", ctypes.c_int, [_vp]),
    ("ndx_event_create", ctypes.c_int, [ctypes.POINTER(_vp), ctypes.c_int]),
    ("ndx_event_destroy", ctypes.c_int, [_vp]),
    ("ndx_event_record", ctypes.c_int, [_vp, _vp]),
    ("ndx_event_query", ctypes.c_int, [_vp]),
    ("ndx_event_synchronize", ctypes.c_int, [_vp]),
    ("ndx_stream_wait_event", ctypes.c_int, [_vp, _vp]),
    ("ndx_event_elapsed_ms", ctypes.c_int, [_vp, _vp, ctypes.POINTER(ctypes.c_float)]),
    ("ndx_malloc_async", ctypes.c_int, [ctypes.POINTER(_vp), _sz, _vp]),
    ("ndx_free_async", ctypes.c_int, [_vp, _vp]),
    ("ndx_memset_async", ctypes.c_int, [_vp, ctypes.c_int, _sz, _vp]),
    ("ndx_host_alloc", ctypes.c_int, [ctypes.POINTER(_vp), _sz]),
    ("ndx_host_free", ctypes.c_int, [_vp]),
    ("ndx_memcpy_h2d_async", ctypes.c_int, [_vp, _vp, _sz, _vp]),
    ("ndx_memcpy_d2h_async", ctypes.c_int, [_vp, _vp, _sz, _vp]),
    ("ndx_memcpy_d2d_async", ctypes.c_int, [_vp, _vp, _sz, _vp]),
    ("ndx_wah_ctl_bytes", _sz, []),
    ("ndx_wah_status_bytes", _sz, [_u64]),
    ("ndx_wah_emit_scratch_bytes", _sz, [_u64]),
    ("ndx_wah_plan", ctypes.c_int, [_vp, _u64, _vp, _vp, _vp]),
    ("ndx_wah_sort", ctypes.c_int, [_vp, _u64, _u32, _vp, _vp, _vp, _vp, _vp]),
    ("ndx_wah_emit", ctypes.c_int, [_vp, _u64, _vp, _vp, _vp, _vp, _vp, _vp]),
    ("ndx_wah_table", ctypes.c_int, [_vp, _vp, _u64, _vp, _vp, _vp]),
    ("ndx_wah_copy_out", ctypes.c_int, [_vp, _vp, _vp, _vp, _vp, _u64, _vp, _u64, _vp]),
    ("ndx_wah_decode_scratch_bytes", _sz, [_u64]),
    ("ndx_wah_decode", ctypes.c_int, [_vp, _u64, _vp, _u64, _vp, _vp, _vp]),
    ("ndx_chunks_and", ctypes.c_int, [_vp, _vp, _vp, _u64, _vp]),
    ("ndx_chunks_or", ctypes.c_int, [_vp, _vp, _vp, _u64, _vp]),
    ("ndx_chunks_andnot", ctypes.c_int, [_vp, _vp, _vp, _u64, _vp]),
    ("ndx_chunks_rows_scratch_bytes", _sz, [_u64]),
    ("ndx_chunks_rows", ctypes.c_int, [_vp, _u64, _u32, _vp, _vp, _vp, _vp]),
    ("ndx_wah_encode_scratch_bytes", _sz, [_u64]),
    ("ndx_wah_encode", ctypes.c_int, [_vp, _u64, ctypes.c_int, _vp, _vp, _vp, _vp]),
    ("ndx_wah_shard_meta", ctypes.c_int, [_vp, _u64, _vp, _vp, _u64, _vp, _vp, _vp]),
    ("ndx_wah_shard_meta_dev", ctypes.c_int, [_vp, _u64, _vp, _vp, _u64, _vp, _vp, _vp]),
    ("ndx_merge_plan_scratch_bytes", _sz, [_u64]),
    ("ndx_merge_plan", ctypes.c_int, [_vp, _u64, _vp, _u32, _vp, _vp, _vp, _vp, _vp]),
    ("ndx_wah_assemble_slots", ctypes.c_int, [_vp, _u32, _vp, _u64, _vp, _vp, _vp]),
    ("ndx_wah_assemble", ctypes.c_int, [_vp, _vp, _u64, _vp, _vp]),
    ("ndx_dist_plan_scratch_bytes", _sz, [_u32, _u64]),
    ("ndx_dist_plan", ctypes.c_int, [_vp, _u64, _vp, _u32, _vp, _vp, _vp, _vp, _vp, _vp]),
    ("ndx_dist_pull", ctypes.c_int, [_vp, _u32, _vp, _u64, _vp, _vp, _u32, ctypes.c_int, _vp, _u64, _u64, _vp]),
    ("ndx_scan_scratch_bytes", _sz, [_u64]),
    ("ndx_scan_exclusive_u32", ctypes.c_int, [_vp, _vp, _u64, _vp, _vp]),
    ("ndx_sort_pairs_scratch_bytes", _sz, [_u64]),
    ("ndx_sort_pairs_u32", ctypes.c_int, [_vp, _vp, _u64, _vp, _vp]),
    ("ndx_compact_prepare", ctypes.c_int, [_vp, _vp, _vp, _u64, _vp, _vp]),
    ("ndx_compact_count", ctypes.c_int, [_vp, _u64, _vp, _vp]),
    ("ndx_compact_move_scratch_bytes", _sz, [_u64]),
    ("ndx_compact_move", ctypes.c_int, [_vp, _vp, _u64, _vp, _vp, _vp, _vp]),
    ("ndx_matmul_f32", ctypes.c_int, [_vp, _vp, _vp, _u64, _vp]),
    ("ndx_tiny_increment", ctypes.c_int, [_vp, _vp]),
]


def lib_path() -> str:
    return os.path.join(_build.LIB, os.environ.get("NDX_LIB", "libndx.so"))


def load() -> ctypes.CDLL:
    """Load libndx.so (building it if absent).  Raises if it cannot load."""
    global _LIB
    if _LIB is None:
        path = lib_path()
        if not os.path.exists(path):
            _build.build_ndx()
        lib = ctypes.CDLL(path)
        for name, rt, args in SIGNATURES:
            fn = getattr(lib, name)
            fn.restype = rt
            fn.argtypes = args
        _LIB = lib
    return _LIB


def check(rc: int, what: str = "") -> None:
    if rc != 0:
        msg = load().ndx_error_string(rc).decode()
        raise NdxError(f"{what}: {msg} ({rc})" if what else f"{msg} ({rc})")


def _ptr(t) -> int:
    return 0 if t is None else int(t.data_ptr())


def _stream_handle(stream) -> int:
    import torch

    s = stream if stream is not None else torch.cuda.current_stream()
    return int(s.cuda_stream)


# ---------------------------------------------------------------------------
# The four-stage WAH build driven directly through the C ABI.  (The C++
# actor runtime in libndactor.so drives the same entry points as compute
# actors; this class is the raw-launch path used for parity tests and as the
# "raw CUDA" side of the dispatch-overhead comparison.)


@dataclass
class HostIndex:
    row_count: int
    entries: np.ndarray  # (D, 3) u32
    words: np.ndarray  # (W,) u32


class WahBuilder:
    """Owns device buffers for builds of up to `capacity` values."""

    def __init__(self, capacity: int = 0, device: int = 0):
        import torch

        self.torch = torch
        self.lib = load()
        check(self.lib.ndx_device_open(device), "device_open")
        self.device = torch.device("cuda", device)
        self.capacity = 0
        if capacity:
            self.ensure(capacity)

    def _alloc(self, nbytes: int, zero: bool = False):
        t = self.torch
        n32 = (nbytes + 3) // 4 + 64
        return (t.zeros if zero else t.empty)(n32, dtype=t.int32, device=self.device)

    def ensure(self, n: int) -> None:
        if n <= self.capacity:
            return
        L = self.lib
        self.ctl = self._alloc(L.ndx_wah_ctl_bytes(), zero=True)
        self.status = self._alloc(L.ndx_wah_status_bytes(n), zero=True)  # zeroed once, statuses only
        self.emit_scr = self._alloc(L.ndx_wah_emit_scratch_bytes(n))
        self.pairs = self._alloc(8 * n)
        self.tmp_pairs = self._alloc(8 * n)
        self.words = self._alloc(8 * n)       # <= 2n words
        self.vstart = self._alloc(4 * n)
        self.values = self._alloc(4 * n)
        self.entries = self._alloc(12 * n)
        self.capacity = n

    def stage_calls(self, keys, n: int, row_base: int = 0, stream=None):
        """The four stage launches as callables (for per-stage timing)."""
        L, s = self.lib, _stream_handle(stream)
        return [
            ("plan", lambda: check(L.ndx_wah_plan(_ptr(keys), n, _ptr(self.ctl), _ptr(self.status), s),
                                   "wah_plan")),
            ("sort", lambda: check(L.ndx_wah_sort(_ptr(keys), n, row_base, _ptr(self.ctl), _ptr(self.pairs),
                                                  _ptr(self.tmp_pairs), _ptr(self.status), s), "wah_sort")),
            ("emit", lambda: check(L.ndx_wah_emit(_ptr(self.pairs), n, _ptr(self.ctl), _ptr(self.words),
                                                  _ptr(self.vstart), _ptr(self.values), _ptr(self.emit_scr), s),
                                   "wah_emit")),
            ("table", lambda: check(L.ndx_wah_table(_ptr(self.values), _ptr(self.vstart), n, _ptr(self.ctl),
                                                    _ptr(self.entries), s), "wah_table")),
        ]

    def launch(self, keys, n: int, row_base: int = 0, stream=None) -> None:
        """Enqueue S1..S4 on `stream` (no host synchronisation)."""
        self.ensure(n)
        if n == 0:
            return
        for _, call in self.stage_calls(keys, n, row_base, stream):
            call()

    def key_range(self) -> tuple[int, int]:
        """(min, max) key of the last build (ndx_wah_counts.min_key/max_key)."""
        c = self.ctl[4:6].cpu().numpy().view(np.uint32)
        return int(c[0]), int(c[1])

    def counts(self) -> tuple[int, int]:
        c = self.ctl[:6].cpu().numpy().view(np.uint64)
        return int(c[0]), int(c[1])

    def fetch(self, n: int) -> HostIndex:
        if n == 0:
            return HostIndex(0, np.zeros((0, 3), np.uint32), np.zeros(0, np.uint32))
        self.torch.cuda.synchronize(self.device)
        W, D = self.counts()
        words = self.words[:W].cpu().numpy().view(np.uint32).copy()
        ent = self.entries[: 3 * D].cpu().numpy().view(np.uint32).reshape(D, 3).copy()
        return HostIndex(n, ent, words)

    def build(self, values: np.ndarray, row_base: int = 0) -> HostIndex:
        """Host array in, host index out (H2D, 4 stages, D2H)."""
        t = self.torch
        v = np.ascontiguousarray(values, dtype=np.uint32)
        n = v.size
        if n == 0:
            return self.fetch(0)
        keys = t.from_numpy(v.view(np.int32)).to(self.device)
        self.launch(keys, n, row_base)
        return self.fetch(n)


# ---------------------------------------------------------------------------
# Primitive wrappers (device tensors in, device tensors out).

class Primitives:
    def __init__(self, device: int = 0):
        import torch

        self.torch = torch
        self.lib = load()
        check(self.lib.ndx_device_open(device), "device_open")
        self.device = torch.device("cuda", device)

    def _dev(self, a: np.ndarray):
        a = np.ascontiguousarray(a, dtype=np.uint32)
        if a.size == 0:
            a = np.zeros(1, np.uint32)
        return self.torch.from_numpy(a.view(np.int32)).to(self.device)

    def _host(self, t, n: int) -> np.ndarray:
        return t[:n].cpu().numpy().view(np.uint32).copy()

    def scan_exclusive(self, x: np.ndarray) -> np.ndarray:
        n = int(np.asarray(x).size)
        if n == 0:
            return np.zeros(0, np.uint32)
        d_in = self._dev(x)
        d_out = self.torch.empty_like(d_in)
        scr = self.torch.zeros(self.lib.ndx_scan_scratch_bytes(n) // 4 + 64, dtype=self.torch.int32,
                               device=self.device)
        check(self.lib.ndx_scan_exclusive_u32(_ptr(d_in), _ptr(d_out), n, _ptr(scr),
                                              _stream_handle(None)), "scan")
        return self._host(d_out, n)

    def sort_pairs(self, keys: np.ndarray, payloads: np.ndarray):
        n = int(np.asarray(keys).size)
        if n == 0:
            return np.zeros(0, np.uint32), np.zeros(0, np.uint32)
        dk, dp = self._dev(keys), self._dev(payloads)
        scr = self.torch.zeros(self.lib.ndx_sort_pairs_scratch_bytes(n) // 4 + 64,
                               dtype=self.torch.int32, device=self.device)
        check(self.lib.ndx_sort_pairs_u32(_ptr(dk), _ptr(dp), n, _ptr(scr),
                                          _stream_handle(None)), "sort_pairs")
        return self._host(dk, n), self._host(dp, n)

    def compact(self, x: np.ndarray) -> np.ndarray:
        """wah::compact (wah_stages.cpp:166-201): split even/odd, prepare ->
        count -> move, read back cfg[1] words."""
        x = np.ascontiguousarray(x, dtype=np.uint32)
        if x.size == 0:
            return np.zeros(0, np.uint32)
        k = (x.size + 1) // 2
        a = np.zeros(k, np.uint32)
        b = np.zeros(k, np.uint32)
        a[: (x.size + 1) // 2] = x[0::2]
        b[: x.size // 2] = x[1::2]
        t, L, s = self.torch, self.lib, _stream_handle(None)
        cfg = self._dev(np.array([k, 0], np.uint32))
        da, db = self._dev(a), self._dev(b)
        inter = t.empty(2 * k, dtype=t.int32, device=self.device)
        tiles = (2 * k + 4095) // 4096
        counts = t.empty(max(tiles, 1), dtype=t.int32, device=self.device)
        out = t.empty(2 * k, dtype=t.int32, device=self.device)
        scr = t.zeros(L.ndx_compact_move_scratch_bytes(2 * k) // 4 + 64, dtype=t.int32,
                      device=self.device)
        check(L.ndx_compact_prepare(_ptr(cfg), _ptr(da), _ptr(db), k, _ptr(inter), s), "prepare")
        check(L.ndx_compact_count(_ptr(inter), 2 * k, _ptr(counts), s), "count")
        check(L.ndx_compact_move(_ptr(cfg), _ptr(inter), 2 * k, _ptr(counts), _ptr(out),
                                 _ptr(scr), s), "move")
        total = int(self._host(cfg, 2)[1])
        return self._host(out, total)
