"""Query side of the index on the GPU.

Decoded bitmaps are chunk arrays: one u32 per 31-row chunk (bit i = row
31c + i), the unit WAH words are made of.  Every operation is one of the
sm_100a kernels behind include/ndx.h; there is no host fallback.

Mirrors the reference's host helpers: decode (p/core/src/wah_words.cpp:21-34),
encode (wah_words.cpp:7-19 + CanonicalWriter, wah.hpp:36-74) and rows_for
(wah_words.cpp:93-103), plus AND / OR / AND-NOT of bitmaps over the index.
"""
from __future__ import annotations

import numpy as np

from . import ndx
from .ndx import _ptr, check

CHUNK = 31


class Query:
    """GPU query kernels on device tensors (int32 views of u32 data)."""

    def __init__(self, device: int = 0):
        import torch
        self.torch = torch
        self.lib = ndx.load()
        self.dev = torch.device("cuda", device)

    def _stream(self):
        return self.torch.cuda.current_stream(self.dev).cuda_stream

    def _scratch(self, nbytes: int):
        return self.torch.empty(nbytes // 4 + 64, dtype=self.torch.int32, device=self.dev)

    def _to_dev(self, a: np.ndarray):
        a = np.ascontiguousarray(a, dtype=np.uint32)
        return self.torch.from_numpy(a.view(np.int32).copy() if a.size else np.zeros(1, np.int32)).to(self.dev)

    # -- decode / encode ------------------------------------------------------
    def decode_chunks(self, d_words, n_words: int, n_chunks: int):
        """Chunk array of n_chunks chunks; returns (chunks, covered)."""
        t = self.torch
        out = t.empty(max(n_chunks, 1), dtype=t.int32, device=self.dev)
        info = t.zeros(4, dtype=t.int32, device=self.dev)
        scr = self._scratch(self.lib.ndx_wah_decode_scratch_bytes(n_words))
        check(self.lib.ndx_wah_decode(_ptr(d_words), n_words, _ptr(out), n_chunks, _ptr(scr), _ptr(info),
                                      self._stream()), "wah_decode")
        inf = info.cpu().numpy().view(np.uint32)
        if inf[1]:
            raise ValueError("fill word with zero length")
        return out[:n_chunks], int(inf[0])

    def decode(self, words: np.ndarray) -> np.ndarray:
        """wah::decode: every covered bit (bool array of 31 * covered)."""
        w = np.ascontiguousarray(words, np.uint32)
        d = self._to_dev(w)
        _, covered = self.decode_chunks(d, w.size, 0)
        chunks, _ = self.decode_chunks(d, w.size, covered)
        return chunks_to_bits(chunks.cpu().numpy().view(np.uint32), covered * CHUNK)

    def encode_chunks(self, d_chunks, n_chunks: int, trim: bool):
        t = self.torch
        words = t.empty(max(n_chunks, 1), dtype=t.int32, device=self.dev)
        info = t.zeros(4, dtype=t.int32, device=self.dev)
        scr = self._scratch(self.lib.ndx_wah_encode_scratch_bytes(n_chunks))
        check(self.lib.ndx_wah_encode(_ptr(d_chunks), n_chunks, int(trim), _ptr(words), _ptr(scr), _ptr(info),
                                      self._stream()), "wah_encode")
        inf = info.cpu().numpy().view(np.uint32)
        if inf[1]:
            raise ValueError("fill longer than the 30-bit length field")
        return words[: int(inf[0])]

    def encode(self, bits) -> np.ndarray:
        """wah::encode: the words cover every bit, rounded up to chunks."""
        b = np.asarray(bits, dtype=bool)
        chunks = bits_to_chunks(b)
        d = self._to_dev(chunks)
        return self.encode_chunks(d, chunks.size, trim=False).cpu().numpy().view(np.uint32).copy()

    # -- bitmap algebra and rows ----------------------------------------------
    def combine(self, op: str, a, b, n_chunks: int):
        t = self.torch
        out = t.empty(max(n_chunks, 1), dtype=t.int32, device=self.dev)
        fn = {"and": self.lib.ndx_chunks_and, "or": self.lib.ndx_chunks_or,
              "andnot": self.lib.ndx_chunks_andnot}[op]
        check(fn(_ptr(a), _ptr(b), _ptr(out), n_chunks, self._stream()), "chunks_" + op)
        return out[:n_chunks]

    def rows(self, d_chunks, n_chunks: int, row_limit: int) -> np.ndarray:
        t = self.torch
        cap = max(int(row_limit), 1)
        rows = t.empty(cap, dtype=t.int32, device=self.dev)
        cnt = t.zeros(1, dtype=t.int32, device=self.dev)
        scr = self._scratch(self.lib.ndx_chunks_rows_scratch_bytes(n_chunks))
        check(self.lib.ndx_chunks_rows(_ptr(d_chunks), n_chunks, row_limit, _ptr(rows), _ptr(scr), _ptr(cnt),
                                       self._stream()), "chunks_rows")
        k = int(cnt.cpu().numpy().view(np.uint32)[0])
        return rows[:k].cpu().numpy().view(np.uint32).copy()


class DeviceIndex:
    """A built index (entries on the host, words on the device) and its
    queries: the bitmap of a value, rows_for, and AND / OR / AND-NOT of two
    values' bitmaps re-encoded as canonical index words."""

    def __init__(self, row_count: int, entries: np.ndarray, d_words, q: Query | None = None):
        self.n = int(row_count)
        self.entries = np.asarray(entries, np.uint32).reshape(-1, 3)
        self.words = d_words
        self.q = q or Query()
        self.n_chunks = (self.n + CHUNK - 1) // CHUNK

    def _entry(self, value: int):
        i = int(np.searchsorted(self.entries[:, 0], np.uint32(value)))
        if i == len(self.entries) or int(self.entries[i, 0]) != value:
            return None
        return self.entries[i]

    def bitmap(self, value: int):
        e = self._entry(value)
        if e is None:
            return self.q.torch.zeros(max(self.n_chunks, 1), dtype=self.q.torch.int32,
                                      device=self.q.dev)[: self.n_chunks]
        off, ln = int(e[1]), int(e[2])
        chunks, _ = self.q.decode_chunks(self.words[off:off + ln], ln, self.n_chunks)
        return chunks

    def rows_for(self, value: int) -> np.ndarray:
        if self._entry(value) is None:
            return np.zeros(0, np.uint32)
        return self.q.rows(self.bitmap(value), self.n_chunks, self.n)

    def combine(self, op: str, a: int, b: int) -> np.ndarray:
        """Canonical words (index form: no trailing fill) of value a OP value b."""
        c = self.q.combine(op, self.bitmap(a), self.bitmap(b), self.n_chunks)
        return self.q.encode_chunks(c, self.n_chunks, trim=True).cpu().numpy().view(np.uint32).copy()


def bits_to_chunks(bits: np.ndarray) -> np.ndarray:
    b = np.asarray(bits, dtype=bool)
    nc = (b.size + CHUNK - 1) // CHUNK
    pad = np.zeros(nc * CHUNK, bool)
    pad[: b.size] = b
    w = (pad.reshape(nc, CHUNK).astype(np.uint64) << np.arange(CHUNK, dtype=np.uint64)).sum(axis=1)
    return w.astype(np.uint32)


def chunks_to_bits(chunks: np.ndarray, nbits: int) -> np.ndarray:
    c = np.asarray(chunks, np.uint32)
    bits = ((c[:, None] >> np.arange(CHUNK, dtype=np.uint32)) & 1).astype(bool).reshape(-1)
    return bits[:nbits]
