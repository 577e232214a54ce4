"""oracle -- TEST INFRASTRUCTURE ONLY (the parity checker, never the product).

Python view of the two CPU checkers built by ``oracle/Makefile``:

* ``Port``      -- ``oracle/wah_oracle.c``, a plain-C restatement of the
                   reference's ``wah::reference_index`` and its helpers
                   (p/core/src/wah_words.cpp:8-103, p/core/include/ndactor/wah.hpp:36-74).
* ``Reference`` -- ``oracle/_ref/libndref.so``, the unmodified reference
                   library compiled from /root/reference (present when it was
                   built in the authoring container; it travels with gpurun).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU legs may
import this module.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
PORT_SO = os.path.join(HERE, "_build", "libwah_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "libndref.so")

_u32p = ctypes.POINTER(ctypes.c_uint32)
_u8p = ctypes.POINTER(ctypes.c_uint8)
_u64p = ctypes.POINTER(ctypes.c_uint64)


def build() -> None:
    """Compile the checkers (C restatement always; reference if present)."""
    subprocess.run(["make", "-s", "-C", HERE, "-j8"], check=True)


def _ptr(a: np.ndarray, t=_u32p):
    return a.ctypes.data_as(t)


@dataclass
class Index:
    """A built WAH index in host memory (mirrors wah::WahIndex, wah.hpp:88-97)."""

    row_count: int
    entries: np.ndarray  # (D, 3) u32: value, offset, length
    words: np.ndarray  # (W,) u32

    def serialize(self) -> bytes:
        """``serialize_index`` (p/core/src/wah_index_io.cpp:30-44)."""
        hdr = np.array([self.row_count, len(self.entries), len(self.words)], "<u4")
        return b"WAH1" + hdr.tobytes() + self.entries.astype("<u4").tobytes() + self.words.astype("<u4").tobytes()

    def digest(self) -> int:
        return Port().digest_parts(self.row_count, self.entries, self.words)

    def __eq__(self, other) -> bool:  # operator==, wah_words.cpp:105-116
        return (
            self.row_count == other.row_count
            and np.array_equal(self.entries, other.entries)
            and np.array_equal(self.words, other.words)
        )


def fnv1a64(data: bytes) -> int:
    """FNV-1a-64 of a short byte string."""
    h = 1469598103934665603
    for b in data:
        h ^= b
        h = (h * 1099511628211) & 0xFFFFFFFFFFFFFFFF
    return h


class Port:
    """The C restatement (oracle/wah_oracle.c)."""

    _lib = None

    def __init__(self):
        if Port._lib is None:
            if not os.path.exists(PORT_SO):
                build()
            lib = ctypes.CDLL(PORT_SO)
            lib.wo_reference_index.restype = ctypes.c_void_p
            lib.wo_reference_index.argtypes = [_u32p, ctypes.c_uint64]
            for name, rt in [
                ("wo_index_row_count", ctypes.c_uint32),
                ("wo_index_num_entries", ctypes.c_uint64),
                ("wo_index_num_words", ctypes.c_uint64),
                ("wo_index_entries", ctypes.c_void_p),
                ("wo_index_words", ctypes.c_void_p),
                ("wo_index_digest", ctypes.c_uint64),
            ]:
                getattr(lib, name).restype = rt
                getattr(lib, name).argtypes = [ctypes.c_void_p]
            lib.wo_index_free.argtypes = [ctypes.c_void_p]
            lib.wo_encode.restype = ctypes.c_uint64
            lib.wo_encode.argtypes = [_u8p, ctypes.c_uint64, _u32p, ctypes.c_uint64]
            lib.wo_decode.restype = ctypes.c_int64
            lib.wo_decode.argtypes = [_u32p, ctypes.c_uint64, _u8p, ctypes.c_uint64]
            lib.wo_decode_exact.restype = ctypes.c_int
            lib.wo_decode_exact.argtypes = [_u32p, ctypes.c_uint64, ctypes.c_uint64, _u8p]
            lib.wo_writer_ops.restype = ctypes.c_uint64
            lib.wo_writer_ops.argtypes = [_u32p, _u64p, ctypes.c_uint64, _u32p, ctypes.c_uint64]
            lib.wo_sort_pairs.argtypes = [_u32p, _u32p, ctypes.c_uint64]
            lib.wo_scan_exclusive.argtypes = [_u32p, _u32p, ctypes.c_uint64]
            lib.wo_filter_nonzero.restype = ctypes.c_uint64
            lib.wo_filter_nonzero.argtypes = [_u32p, ctypes.c_uint64, _u32p]
            lib.wo_rows_for.restype = ctypes.c_uint64
            lib.wo_rows_for.argtypes = [ctypes.c_void_p, ctypes.c_uint32, _u32p, ctypes.c_uint64]
            lib.wo_digest_parts.restype = ctypes.c_uint64
            lib.wo_digest_parts.argtypes = [ctypes.c_uint32, _u32p, ctypes.c_uint64, _u32p, ctypes.c_uint64]
            Port._lib = lib
        self.lib = Port._lib

    # -- index -------------------------------------------------------------
    def reference_index(self, values: np.ndarray) -> Index:
        v = np.ascontiguousarray(values, dtype=np.uint32)
        h = self.lib.wo_reference_index(_ptr(v), v.size)
        try:
            return self._take(h)
        finally:
            self.lib.wo_index_free(h)

    def _take(self, h) -> Index:
        L = self.lib
        d, w = L.wo_index_num_entries(h), L.wo_index_num_words(h)
        ent = np.zeros((d, 3), np.uint32)
        wor = np.zeros(w, np.uint32)
        if d:
            ctypes.memmove(ent.ctypes.data, L.wo_index_entries(h), d * 12)
        if w:
            ctypes.memmove(wor.ctypes.data, L.wo_index_words(h), w * 4)
        return Index(int(L.wo_index_row_count(h)), ent, wor)

    def digest_of(self, values: np.ndarray) -> int:
        v = np.ascontiguousarray(values, dtype=np.uint32)
        h = self.lib.wo_reference_index(_ptr(v), v.size)
        try:
            return int(self.lib.wo_index_digest(h))
        finally:
            self.lib.wo_index_free(h)

    def rows_for(self, values: np.ndarray, value: int) -> np.ndarray:
        v = np.ascontiguousarray(values, dtype=np.uint32)
        h = self.lib.wo_reference_index(_ptr(v), v.size)
        try:
            n = self.lib.wo_rows_for(h, value, None, 0)
            out = np.zeros(max(n, 1), np.uint32)
            self.lib.wo_rows_for(h, value, _ptr(out), n)
            return out[:n]
        finally:
            self.lib.wo_index_free(h)

    def digest_parts(self, row_count: int, entries: np.ndarray, words: np.ndarray) -> int:
        e = np.ascontiguousarray(entries, dtype=np.uint32).reshape(-1)
        w = np.ascontiguousarray(words, dtype=np.uint32)
        e_ = e if e.size else np.zeros(1, np.uint32)
        w_ = w if w.size else np.zeros(1, np.uint32)
        return int(self.lib.wo_digest_parts(row_count, _ptr(e_), e.size // 3, _ptr(w_), w.size))

    # -- words ---------------------------------------------------------------
    def encode(self, bits) -> np.ndarray:
        b = np.ascontiguousarray(np.asarray(bits, dtype=np.uint8))
        b_ = b if b.size else np.zeros(1, np.uint8)
        n = self.lib.wo_encode(_ptr(b_, _u8p), b.size, None, 0)
        out = np.zeros(max(n, 1), np.uint32)
        self.lib.wo_encode(_ptr(b_, _u8p), b.size, _ptr(out), n)
        return out[:n]

    def decode(self, words) -> np.ndarray:
        w = np.ascontiguousarray(np.asarray(words, dtype=np.uint32))
        w_ = w if w.size else np.zeros(1, np.uint32)
        n = self.lib.wo_decode(_ptr(w_), w.size, None, 0)
        if n < 0:
            raise ValueError("fill word with zero length")
        out = np.zeros(max(n, 1), np.uint8)
        self.lib.wo_decode(_ptr(w_), w.size, _ptr(out, _u8p), n)
        return out[:n]

    def decode_exact(self, words, n: int) -> np.ndarray:
        w = np.ascontiguousarray(np.asarray(words, dtype=np.uint32))
        w_ = w if w.size else np.zeros(1, np.uint32)
        out = np.zeros(max(n, 1), np.uint8)
        rc = self.lib.wo_decode_exact(_ptr(w_), w.size, n, _ptr(out, _u8p))
        if rc:
            raise ValueError(
                {1: "fill word with zero length", 2: "words cover fewer bits than expected",
                 3: "words cover a whole chunk beyond the expected bits", 4: "padding bit is set"}[rc])
        return out[:n]

    def writer(self, ops) -> np.ndarray:
        """ops: list of ("chunk", bits) | ("uniform", ones, count)."""
        kinds, args = [], []
        for op in ops:
            if op[0] == "chunk":
                kinds.append(0)
                args.append(op[1])
            else:
                kinds.append(2 if op[1] else 1)
                args.append(op[2])
        k = np.array(kinds, np.uint32)
        a = np.array(args, np.uint64)
        n = self.lib.wo_writer_ops(_ptr(k), _ptr(a, _u64p), len(kinds), None, 0)
        out = np.zeros(max(n, 1), np.uint32)
        self.lib.wo_writer_ops(_ptr(k), _ptr(a, _u64p), len(kinds), _ptr(out), n)
        return out[:n]

    # -- device-primitive oracles ---------------------------------------------
    def sort_pairs(self, keys, payloads):
        k = np.array(keys, dtype=np.uint32, copy=True)
        p = np.array(payloads, dtype=np.uint32, copy=True)
        if k.size:
            self.lib.wo_sort_pairs(_ptr(k), _ptr(p), k.size)
        return k, p

    def scan_exclusive(self, x) -> np.ndarray:
        x = np.ascontiguousarray(x, dtype=np.uint32)
        out = np.zeros_like(x)
        if x.size:
            self.lib.wo_scan_exclusive(_ptr(x), _ptr(out), x.size)
        return out

    def filter_nonzero(self, x) -> np.ndarray:
        x = np.ascontiguousarray(x, dtype=np.uint32)
        out = np.zeros(max(x.size, 1), np.uint32)
        m = self.lib.wo_filter_nonzero(_ptr(x if x.size else out), x.size, _ptr(out))
        return out[:m]


class Reference:
    """The unmodified reference library (oracle/_ref/libndref.so)."""

    _lib = None

    @staticmethod
    def available() -> bool:
        return os.path.exists(REF_SO)

    def __init__(self):
        if Reference._lib is None:
            if not os.path.exists(REF_SO):
                raise FileNotFoundError(REF_SO + " (build with make -C oracle)")
            lib = ctypes.CDLL(REF_SO)
            lib.ref_reference_index.restype = ctypes.c_void_p
            lib.ref_reference_index.argtypes = [_u32p, ctypes.c_uint64]
            lib.ref_build_index_sim.restype = ctypes.c_void_p
            lib.ref_build_index_sim.argtypes = [_u32p, ctypes.c_uint64, ctypes.c_uint, ctypes.c_uint]
            for name, rt in [("ref_index_row_count", ctypes.c_uint32),
                             ("ref_index_num_entries", ctypes.c_uint64),
                             ("ref_index_num_words", ctypes.c_uint64),
                             ("ref_index_digest", ctypes.c_uint64)]:
                getattr(lib, name).restype = rt
                getattr(lib, name).argtypes = [ctypes.c_void_p]
            lib.ref_index_entries.argtypes = [ctypes.c_void_p, _u32p]
            lib.ref_index_words.argtypes = [ctypes.c_void_p, _u32p]
            lib.ref_index_free.argtypes = [ctypes.c_void_p]
            lib.ref_compact_sim.restype = ctypes.c_uint64
            lib.ref_compact_sim.argtypes = [_u32p, ctypes.c_uint64, _u32p]
            lib.ref_gen_uniform.argtypes = [ctypes.c_uint32, ctypes.c_uint64, ctypes.c_uint32, _u32p]
            lib.ref_gen_zipf.argtypes = [ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint32, ctypes.c_double, _u32p]
            Reference._lib = lib
        self.lib = Reference._lib

    def _take(self, h) -> Index:
        L = self.lib
        d, w = L.ref_index_num_entries(h), L.ref_index_num_words(h)
        ent = np.zeros((d, 3), np.uint32)
        wor = np.zeros(w, np.uint32)
        if d:
            L.ref_index_entries(h, _ptr(ent))
        if w:
            L.ref_index_words(h, _ptr(wor))
        return Index(int(L.ref_index_row_count(h)), ent, wor)

    def reference_index(self, values) -> Index:
        v = np.ascontiguousarray(values, dtype=np.uint32)
        v_ = v if v.size else np.zeros(1, np.uint32)
        h = self.lib.ref_reference_index(_ptr(v_), v.size)
        try:
            return self._take(h)
        finally:
            self.lib.ref_index_free(h)

    def digest_of(self, values) -> int:
        v = np.ascontiguousarray(values, dtype=np.uint32)
        v_ = v if v.size else np.zeros(1, np.uint32)
        h = self.lib.ref_reference_index(_ptr(v_), v.size)
        try:
            return int(self.lib.ref_index_digest(h))
        finally:
            self.lib.ref_index_free(h)

    def build_index_sim(self, values, cus: int, digit_bits: int = 8) -> Index:
        v = np.ascontiguousarray(values, dtype=np.uint32)
        v_ = v if v.size else np.zeros(1, np.uint32)
        h = self.lib.ref_build_index_sim(_ptr(v_), v.size, cus, digit_bits)
        try:
            return self._take(h)
        finally:
            self.lib.ref_index_free(h)

    def compact_sim(self, x) -> np.ndarray:
        x = np.ascontiguousarray(x, dtype=np.uint32)
        out = np.zeros(max(x.size, 1), np.uint32)
        m = self.lib.ref_compact_sim(_ptr(x if x.size else out), x.size, _ptr(out))
        return out[:m]

    def gen_uniform(self, seed: int, n: int, card: int) -> np.ndarray:
        out = np.zeros(max(n, 1), np.uint32)
        self.lib.ref_gen_uniform(seed, n, card, _ptr(out))
        return out[:n]

    def gen_zipf(self, seed: int, n: int, k: int, s: float = 1.0) -> np.ndarray:
        out = np.zeros(max(n, 1), np.uint32)
        self.lib.ref_gen_zipf(seed, n, k, s, _ptr(out))
        return out[:n]
