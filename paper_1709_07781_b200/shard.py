"""Multi-GPU WAH build: row shards, metadata exchange, boundary merge.

SURVEY.md 8(e) / Appendix B.  One process per GPU (torch.distributed; NCCL on
GPUs, gloo for the CPU tests).  Rank g builds rows [S_g, S_{g+1}) of the
global column with global row ids (S_g a multiple of 31, so no chunk
straddles two ranks), then:

  1. ndx_wah_shard_meta: per value (value, first/last chunk, ones-fill
     lengths at both ends of the body, body range) -- 32 B per value;
  2. all-gather of the metadata (<= 8 x 65,536 x 32 B = 16 MB);
  3. every rank plans the merge over the metadata (ndactor_merge_plan, host
     C++, replicated): merged (value, offset, length) table and, per local
     value, where its words go and which end words change;
  4. the words are gathered to rank 0 (point-to-point over NVLink) and
     ndx_wah_assemble copies every piece into place; or (exchange_owned)
     one all-to-all-v by value-range ownership leaves every rank a
     contiguous slice of the merged word array.

The result on rank 0 is bit-identical to a single-device build of the whole
column.  No data-path work runs on the host: step 3 touches only metadata.
"""
from __future__ import annotations

import ctypes

import numpy as np

from . import runtime as _rt

META_DTYPE = np.dtype([("value", "<u4"), ("f", "<u4"), ("l", "<u4"), ("a", "<u4"), ("z", "<u4"),
                       ("body_off", "<u4"), ("body_len", "<u4"), ("skip", "<u4")])
PIECE_DTYPE = np.dtype([("dst", "<u8"), ("src_off", "<u4"), ("src_len", "<u4"), ("lead", "<u4"),
                        ("pad", "<u4")])
assert META_DTYPE.itemsize == 32 and PIECE_DTYPE.itemsize == 24


def shard_bounds(n: int, shards: int) -> np.ndarray:
    """S_0..S_G: inner bounds multiples of 31, chunk counts balanced."""
    lib = _rt.load()
    out = np.zeros(shards + 1, np.uint64)
    _rt._check(lib.ndactor_shard_bounds(n, shards, out.ctypes.data), "shard_bounds")
    return out


_SCRATCH: dict = {}


def _scratch(name: str, n: int, dtype) -> np.ndarray:
    """Reused host buffers (fresh pages cost a fault each on first touch).
    Results returned by plan_merge are views that stay valid until the next
    call of the same process."""
    a = _SCRATCH.get(name)
    if a is None or a.size < n or a.dtype != np.dtype(dtype):
        a = np.empty(max(n, 1), dtype)
        a.view(np.uint8)[:] = 0  # touch the pages once
        _SCRATCH[name] = a
    return a[:n]


def plan_merge(metas, sizes=None):
    """Merge plan over per-shard metadata (META_DTYPE, ascending values).

    `metas` is a list of per-shard arrays, or a padded (G, cap) array with
    `sizes` giving each shard's record count (no copy).  Returns (entries
    (D,3) u32, pieces list per shard (PIECE_DTYPE, dst absolute), words);
    the arrays are views of reused buffers (copy them to keep them across
    calls)."""
    lib = _rt.load()
    if sizes is None:
        counts = np.array([m.size for m in metas], np.uint64)
        cat = np.ascontiguousarray(np.concatenate(metas) if len(metas) else np.zeros(0, META_DTYPE), META_DTYPE)
        stride = 0
        G = len(metas)
    else:
        cat = np.ascontiguousarray(metas)
        G, stride = cat.shape
        counts = np.asarray(sizes, np.uint64)
    total = int(counts.sum())
    entries = _scratch("entries", max(total, 1) * 3, np.uint32).reshape(-1, 3)
    pieces = _scratch("pieces", max(cat.size, 1), PIECE_DTYPE)
    ne, nw = ctypes.c_uint64(), ctypes.c_uint64()
    _rt._check(lib.ndactor_merge_plan(G, cat.ctypes.data, counts.ctypes.data, stride, entries.ctypes.data,
                                      pieces.ctypes.data, ctypes.byref(ne), ctypes.byref(nw)), "merge_plan")
    out, off = [], 0
    for g, c in enumerate(counts.tolist()):
        at = g * stride if stride else off
        out.append(pieces[at:at + c])
        off += c
    return entries[: ne.value], out, int(nw.value)


# ---------------------------------------------------------------------------
# Collectives (torch.distributed; tensors on the backend's device)

def _dev_for(group=None):
    import torch.distributed as dist
    return "cuda" if dist.get_backend(group) == "nccl" else "cpu"


def exchange_meta(meta: np.ndarray, group=None) -> list[np.ndarray]:
    """All-gather every rank's metadata (variable length)."""
    import torch
    import torch.distributed as dist
    dev = _dev_for(group)
    ws = dist.get_world_size(group)
    cnt = torch.tensor([meta.size], dtype=torch.int64, device=dev)
    cnts = [torch.zeros(1, dtype=torch.int64, device=dev) for _ in range(ws)]
    dist.all_gather(cnts, cnt, group=group)
    sizes = [int(c.item()) for c in cnts]
    cap = max(max(sizes), 1)
    buf = np.zeros(cap, META_DTYPE)
    buf[: meta.size] = meta
    t = torch.from_numpy(buf.view(np.int32).copy()).to(dev)
    outs = [torch.zeros_like(t) for _ in range(ws)]
    dist.all_gather(outs, t, group=group)
    return [o.cpu().numpy().view(META_DTYPE)[:s].copy() for o, s in zip(outs, sizes)]


def exchange_meta_device(meta_d, D: int, group=None):
    """All-gather of device-resident metadata (meta_d: int32 tensor of at
    least D*8 words on this rank's GPU) over NCCL.  Returns (a (G, cap*8)
    int32 device tensor of the padded records, per-rank record counts): the
    input of plan_merge_device; `host_metas` turns it into the (G, cap)
    META_DTYPE array plan_merge takes."""
    import torch
    import torch.distributed as dist
    ws = dist.get_world_size(group)
    dev = meta_d.device
    cnt = torch.tensor([D], dtype=torch.int64, device=dev)
    cnts = torch.empty(ws, dtype=torch.int64, device=dev)
    dist.all_gather_into_tensor(cnts, cnt, group=group)
    sizes = cnts.cpu().tolist()
    cap = max(max(sizes), 1)
    if meta_d.numel() >= cap * 8:
        mine = meta_d[: cap * 8]
    else:
        mine = torch.zeros(cap * 8, dtype=torch.int32, device=dev)
        mine[: D * 8] = meta_d[: D * 8]
    out = torch.empty(ws * cap * 8, dtype=torch.int32, device=dev)
    dist.all_gather_into_tensor(out, mine.contiguous(), group=group)
    return out.view(ws, cap * 8), sizes


def host_metas(padded) -> np.ndarray:
    g = padded.shape[0]
    return padded.cpu().numpy().view(META_DTYPE).reshape(g, -1)


def plan_merge_device(padded, sizes):
    """The merge plan on the GPU (ndx_merge_plan), same result as plan_merge.
    padded: (G, cap*8) int32 device tensor; returns (entries (D,3) int32
    device tensor, pieces (G*cap*24 bytes) device tensor, D, W)."""
    import torch
    from . import ndx
    lib = ndx.load()
    G, cap8 = padded.shape
    cap = cap8 // 8
    counts = np.asarray(sizes, np.uint64)
    dev = padded.device
    rec = int(counts.sum())
    entries = torch.empty(max(rec, 1) * 3, dtype=torch.int32, device=dev)
    pieces = torch.empty(max(G * cap, 1) * 6, dtype=torch.int32, device=dev)
    totals = torch.zeros(3, dtype=torch.int64, device=dev)
    scr = torch.empty(lib.ndx_merge_plan_scratch_bytes(rec) // 4 + 64, dtype=torch.int32, device=dev)
    ndx.check(lib.ndx_merge_plan(ndx._ptr(padded), cap, counts.ctypes.data, G, ndx._ptr(entries), ndx._ptr(pieces),
                                 ndx._ptr(totals), ndx._ptr(scr), torch.cuda.current_stream(dev).cuda_stream),
              "merge_plan")
    t = totals.cpu().numpy()
    if t[2]:
        raise RuntimeError("merge plan: inconsistent shard metadata (flags %d)" % int(t[2]))
    D, W = int(t[0]), int(t[1])
    return entries[: 3 * D].view(D, 3), pieces, D, W


def assemble_slots(staged: list, pieces, cap: int, sizes, total_words: int, out=None):
    """Assemble from a device plan: staged[g] = shard g's words (device)."""
    import torch
    from . import ndx
    lib = ndx.load()
    dev = pieces.device
    if out is None:
        out = torch.empty(max(total_words, 1), dtype=torch.int32, device=dev)
    srcs = (ctypes.c_void_p * len(staged))(*[s.data_ptr() for s in staged])
    counts = np.asarray(sizes, np.uint64)
    ndx.check(lib.ndx_wah_assemble_slots(srcs, len(staged), ndx._ptr(pieces), cap, counts.ctypes.data,
                                         ndx._ptr(out), torch.cuda.current_stream(dev).cuda_stream),
              "assemble_slots")
    return out[:total_words]


def gather_words(words, dst: int = 0, group=None):
    """Point-to-point gather of every rank's local words (a 1-D int32 tensor
    on the backend's device) to `dst`; returns the list on dst, None elsewhere."""
    import torch
    import torch.distributed as dist
    rank, ws = dist.get_rank(group), dist.get_world_size(group)
    dev = words.device
    n = torch.tensor([words.numel()], dtype=torch.int64, device=dev)
    ns = [torch.zeros(1, dtype=torch.int64, device=dev) for _ in range(ws)]
    dist.all_gather(ns, n, group=group)
    if rank != dst:
        if words.numel():
            dist.send(words.contiguous(), dst, group=group)
        return None
    out = []
    for g in range(ws):
        k = int(ns[g].item())
        if g == rank:
            out.append(words)
        else:
            buf = torch.empty(k, dtype=words.dtype, device=dev)
            if k:
                dist.recv(buf, g, group=group)
            out.append(buf)
    return out


# ---------------------------------------------------------------------------
# GPU path

class ShardBuilder:
    """Local build of one shard on this rank's GPU + its metadata."""

    def __init__(self, capacity: int = 0, device: int = 0):
        from . import ndx
        self.ndx = ndx
        self.b = ndx.WahBuilder(capacity, device)
        self.torch = self.b.torch

    def build(self, keys, n: int, row_base: int):
        """keys: device int32 tensor (n values).  Returns (W, D, meta device
        tensor) after the four stages and the metadata kernel."""
        t, ndx = self.torch, self.ndx
        self.b.launch(keys, n, row_base)
        W, D = self.b.counts()
        meta = t.empty(max(D, 1) * 8, dtype=t.int32, device=keys.device)
        ndx.check(self.b.lib.ndx_wah_shard_meta(ndx._ptr(self.b.pairs), n, ndx._ptr(self.b.ctl),
                                               ndx._ptr(self.b.entries), D,
                                               ndx._ptr(self.b.words), ndx._ptr(meta),
                                               t.cuda.current_stream().cuda_stream), "shard_meta")
        return W, D, meta

    @property
    def words(self):
        return self.b.words


def split_pieces(p: np.ndarray, block: int = 4096) -> np.ndarray:
    """Cut pieces into runs of at most `block` words so the copy spreads over
    the whole GPU (a hot value's piece can hold tens of millions of words)."""
    if p.size == 0:
        return p
    body = p["src_len"].astype(np.int64)
    nb = np.maximum(1, (body + block - 1) // block)
    if int(nb.max()) == 1:
        return p
    idx = np.repeat(np.arange(p.size), nb)
    first = np.concatenate([[0], np.cumsum(nb)[:-1]])
    k = np.arange(idx.size) - np.repeat(first, nb)  # block index inside its piece
    out = np.zeros(idx.size, PIECE_DTYPE)
    lead = p["lead"][idx]
    has_lead = (lead != 0).astype(np.int64)
    out["src_off"] = (p["src_off"][idx].astype(np.int64) + k * block).astype(np.uint32)
    out["src_len"] = np.minimum(block, body[idx] - k * block).astype(np.uint32)
    out["lead"] = np.where(k == 0, lead, 0)
    out["dst"] = (p["dst"][idx].astype(np.int64) + np.where(k == 0, 0, has_lead + k * block)).astype(np.uint64)
    return out


def assemble(staged: list, pieces: list[np.ndarray], total_words: int, device, out=None):
    """Copy every shard's pieces into the merged word array on `device`
    (ndx_wah_assemble).  staged[g]: shard g's local words (device int32).
    With only some shards' pieces, only their positions of `out` are written
    (a rank putting its own pieces into final form)."""
    import torch
    from . import ndx
    lib = ndx.load()
    sizes = [int(s.numel()) for s in staged]
    base = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
    if len(staged) == 1:
        src = staged[0].reshape(-1)
    else:
        src = torch.cat([s.reshape(-1) for s in staged]) if staged else torch.zeros(0, dtype=torch.int32,
                                                                                   device=device)
    allp = []
    for g, p in enumerate(pieces):
        q = p.copy()
        q["src_off"] = (q["src_off"].astype(np.int64) + base[g]).astype(np.uint32)
        allp.append(q)
    cat = split_pieces(np.concatenate(allp) if allp else np.zeros(0, PIECE_DTYPE))
    if base[-1] >= 2 ** 32:
        raise ValueError("staged words exceed u32 offsets")
    pd = torch.from_numpy(cat.view(np.uint8).copy()).to(device)
    if out is None:
        out = torch.empty(max(total_words, 1), dtype=torch.int32, device=device)
    ndx.check(lib.ndx_wah_assemble(ndx._ptr(src), ndx._ptr(pd), cat.size, ndx._ptr(out),
                                   torch.cuda.current_stream().cuda_stream), "assemble")
    return out[:total_words]


# ---------------------------------------------------------------------------
# Owned slices: all-to-all-v by value range

def owner_bounds(entries: np.ndarray, total_words: int, shards: int) -> np.ndarray:
    """Word bounds b_0..b_G of the slices each rank owns, cut at value
    boundaries: b_h = offset of the first value whose offset >= h*W/G.  Every
    piece is one value's words from one shard, so no piece straddles a cut.
    entries: merged (D,3) u32 table (replicated on every rank)."""
    off = np.asarray(entries, np.uint32).reshape(-1, 3)[:, 1].astype(np.int64)
    want = (np.arange(shards + 1, dtype=np.int64) * total_words) // max(shards, 1)
    idx = np.searchsorted(off, want[1:-1], side="left")
    inner = np.where(idx < off.size, off[np.minimum(idx, max(off.size - 1, 0))] if off.size else 0, total_words)
    return np.concatenate([[0], inner, [total_words]]).astype(np.int64)


def owned_plan(pieces: list[np.ndarray], bounds: np.ndarray, rank: int):
    """Host plan of the all-to-all-v, from the replicated merge plan only.

    Returns (pack, send_counts, place, recv_counts):
      pack   -- this rank's pieces with dst rewritten to packed positions: the
                assembly writes this rank's final-form words (lead words
                included) contiguously in global order, i.e. grouped by owner;
      send_counts[h] -- words of that packed buffer owned by rank h;
      place  -- pure copies (lead 0) from the received buffer (sources
                concatenated in rank order) to positions inside the owned
                slice [bounds[rank], bounds[rank+1]);
      recv_counts[g] -- words rank g sends here."""
    G = len(pieces)
    send_counts = np.zeros((G, G), np.int64)  # [src, dst]
    ranges = []
    for g, p in enumerate(pieces):
        a = np.ascontiguousarray(p).view(np.uint32).reshape(-1, 6)  # dst lo, dst hi, off, len, lead, pad
        dst = a[:, 0].astype(np.int64) | (a[:, 1].astype(np.int64) << 32)
        pl = a[:, 3].astype(np.int64) + (a[:, 4] != 0)
        own = np.searchsorted(bounds, dst, side="right") - 1
        if a.shape[0] and (np.any(np.diff(dst) < 0) or own[0] < 0 or np.any(dst + pl > bounds[np.minimum(own + 1, G)])):
            raise ValueError("owned_plan: pieces out of order or straddling an owner bound")
        cum = np.concatenate([[0], np.cumsum(pl)])
        cut = np.searchsorted(own, np.arange(G + 1), side="left")  # owners ascend with dst
        send_counts[g] = np.diff(cum[cut])
        if g == rank:
            pack = np.ascontiguousarray(p).copy()
            pack["dst"] = cum[:-1].astype(np.uint64)
        lo, hi = int(cut[rank]), int(cut[rank + 1])
        ranges.append((dst[lo:hi], pl[lo:hi]))
    recv_counts = send_counts[:, rank].copy()
    dst = np.concatenate([r[0] for r in ranges]) if G else np.zeros(0, np.int64)
    k = np.concatenate([r[1] for r in ranges]) if G else np.zeros(0, np.int64)
    keep = k > 0
    off = np.cumsum(k) - k  # sources concatenated in rank order
    place = np.zeros(int(keep.sum()), PIECE_DTYPE)
    place["src_off"] = off[keep].astype(np.uint32)
    place["src_len"] = k[keep].astype(np.uint32)
    place["dst"] = (dst[keep] - bounds[rank]).astype(np.uint64)
    return pack, send_counts[rank].copy(), place, recv_counts


def alltoallv_words(send, send_counts, recv_counts, group=None):
    """One all_to_all_single with per-rank split sizes (NCCL over NVLink on
    GPUs, gloo on CPU)."""
    import torch
    import torch.distributed as dist
    out = torch.empty(int(np.sum(recv_counts)), dtype=send.dtype, device=send.device)
    dist.all_to_all_single(out, send.contiguous(), output_split_sizes=[int(x) for x in recv_counts],
                           input_split_sizes=[int(x) for x in send_counts], group=group)
    return out


def exchange_owned(words_local, entries: np.ndarray, pieces: list[np.ndarray], total_words: int, group=None):
    """SURVEY.md 8(e) step 3 on the GPU: pack this rank's final-form words
    (ndx_wah_assemble), all-to-all-v them by value-range ownership, place the
    received runs (ndx_wah_assemble).  Returns (bounds, slice): this rank's
    contiguous slice [bounds[r], bounds[r+1]) of the merged word array."""
    import torch.distributed as dist
    rank, G = dist.get_rank(group), dist.get_world_size(group)
    bounds = owner_bounds(entries, total_words, G)
    pack, sc, place, rc = owned_plan(pieces, bounds, rank)
    dev = words_local.device
    send = assemble([words_local], [pack], int(sc.sum()), dev)
    recv = alltoallv_words(send, sc, rc, group)
    mine = int(bounds[rank + 1] - bounds[rank])
    return bounds, assemble([recv], [place], mine, dev)


def build_distributed(values_local: np.ndarray, row_base: int, builder: ShardBuilder, group=None,
                      owned: bool = False):
    """The whole multi-GPU build for this rank's shard (one process per GPU).

    Returns (entries (D,3) u32 numpy, words device tensor) on rank 0 and
    (entries, None) elsewhere; entries are replicated on every rank.  With
    owned=True every rank instead gets (entries, (bounds, slice)): its
    contiguous value-range slice of the merged words (exchange_owned)."""
    import torch
    import torch.distributed as dist
    dev = torch.device("cuda", torch.cuda.current_device())
    keys = torch.from_numpy(np.ascontiguousarray(values_local, np.uint32).view(np.int32)).to(dev)
    n = keys.numel()
    W, D, meta_d = builder.build(keys, n, row_base)
    padded, sizes = exchange_meta_device(meta_d, D, group)
    entries, pieces, _, total = plan_merge_device(padded, sizes)
    if owned:
        G, cap = padded.shape[0], padded.shape[1] // 8
        hp = pieces.cpu().numpy().view(PIECE_DTYPE)[: G * cap].reshape(G, cap)
        ent = entries.cpu().numpy().view(np.uint32)
        plist = [hp[g, : int(sizes[g])].copy() for g in range(G)]
        return ent, exchange_owned(builder.words[:W], ent, plist, total, group)
    staged = gather_words(builder.words[:W], dst=0, group=group)
    ent = entries.cpu().numpy().view(np.uint32)
    if dist.get_rank(group) != 0:
        return ent, None
    return ent, assemble_slots(staged, pieces, padded.shape[1] // 8, sizes, total)
