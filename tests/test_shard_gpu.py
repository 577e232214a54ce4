"""Multi-GPU build kernels on one GPU: the shards are built one after the
other (no rank waits on another), then ndx_wah_shard_meta, the merge plan
and ndx_wah_assemble must give the single-device index bit for bit."""
import numpy as np
import pytest

from paper_1709_07781_b200 import gen, shard
from tests import shard_helpers as H

pytestmark = pytest.mark.gpu


def _sharded_build(v: np.ndarray, g: int):
    import torch

    sb = shard.ShardBuilder(1 << 16)
    b = shard.shard_bounds(v.size, g).astype(np.int64)
    metas, staged = [], []
    for k in range(g):
        part = v[b[k]:b[k + 1]]
        if part.size == 0:
            metas.append(np.zeros(0, shard.META_DTYPE))
            staged.append(torch.zeros(0, dtype=torch.int32, device="cuda"))
            continue
        keys = torch.from_numpy(part.view(np.int32).copy()).cuda()
        W, D, meta = sb.build(keys, part.size, int(b[k]))
        metas.append(meta[: D * 8].cpu().numpy().view(shard.META_DTYPE).copy())
        staged.append(sb.words[:W].clone())
    entries, pieces, total = shard.plan_merge(metas)
    words = shard.assemble(staged, pieces, total, torch.device("cuda"))
    # the device planner from the same metadata, padded as the all-gather delivers it
    cap = max([m.size for m in metas] + [1])
    pad = np.zeros((g, cap), shard.META_DTYPE)
    for k, m in enumerate(metas):
        pad[k, :m.size] = m
    dpad = torch.from_numpy(pad.view(np.int32).reshape(g, cap * 8).copy()).cuda()
    d_ent, d_pieces, nent, total2 = shard.plan_merge_device(dpad, [m.size for m in metas])
    assert total2 == total and np.array_equal(d_ent.cpu().numpy().view(np.uint32), entries)
    words2 = shard.assemble_slots(staged, d_pieces, cap, [m.size for m in metas], total2)
    assert np.array_equal(words2.cpu().numpy(), words.cpu().numpy())
    return entries, words.cpu().numpy().view(np.uint32)


@pytest.mark.parametrize("g", [2, 3, 8])
@pytest.mark.parametrize("name", sorted(H.columns()))
def test_sharded_build_matches_single_device(port, name, g):
    v = H.columns()[name]
    entries, words = _sharded_build(v, g)
    ref = port.reference_index(v)
    assert np.array_equal(entries, ref.entries) and np.array_equal(words, ref.words), (name, g)


def test_shard_meta_kernel_matches_host(port):
    import torch

    v = H.columns()["hot_cold"]
    sb = shard.ShardBuilder(1 << 16)
    base = 31 * 1000
    W, D, meta = sb.build(torch.from_numpy(v.view(np.int32).copy()).cuda(), v.size, base)
    got = meta[: D * 8].cpu().numpy().view(shard.META_DTYPE)
    e, w = H.local_index(port, v, base)
    assert np.array_equal(got, H.local_meta(v, base, e, w))


@pytest.mark.parametrize("g", [2, 4, 8])
def test_sharded_zipf_digest(port, g):
    """2^22 Zipf values (the C4 distribution) over g shards: digest of the
    merged index equals the reference's."""
    v = gen.zipf(42, 1 << 22, 65536, 1.0)
    entries, words = _sharded_build(v, g)
    assert port.digest_parts(v.size, entries, words) == port.digest_of(v)


@pytest.mark.parametrize("g", [2, 3, 8])
@pytest.mark.parametrize("name", ["hot_cold", "ones_across", "ones_tiny_shards", "blocks"])
def test_owned_slices_on_gpu(port, name, g):
    """All-to-all-v by value range with the device
    kernels: each shard packs its final-form words (ndx_wah_assemble), the
    exchange is simulated by slicing the packed buffers, each owner places
    its runs (ndx_wah_assemble).  The slices tile the reference index."""
    import torch

    v = H.columns()[name]
    sb = shard.ShardBuilder(1 << 16)
    b = shard.shard_bounds(v.size, g).astype(np.int64)
    metas, staged = [], []
    for k in range(g):
        part = v[b[k]:b[k + 1]]
        if part.size == 0:  # more shards than chunks: an empty shard sends nothing
            metas.append(np.zeros(0, shard.META_DTYPE))
            staged.append(torch.zeros(0, dtype=torch.int32, device="cuda"))
            continue
        keys = torch.from_numpy(part.view(np.int32).copy()).cuda()
        W, D, meta = sb.build(keys, part.size, int(b[k]))
        metas.append(meta[: D * 8].cpu().numpy().view(shard.META_DTYPE).copy())
        staged.append(sb.words[:W].clone())
    entries, pieces, total = shard.plan_merge(metas)
    entries, pieces = entries.copy(), [p.copy() for p in pieces]
    bounds = shard.owner_bounds(entries, total, g)
    plans = [shard.owned_plan(pieces, bounds, r) for r in range(g)]
    sends = []
    for r, (pack, sc, place, rc) in enumerate(plans):
        buf = shard.assemble([staged[r]], [pack], int(sc.sum()), torch.device("cuda"))
        sends.append(torch.split(buf, [int(x) for x in sc]))
    out = []
    for r, (pack, sc, place, rc) in enumerate(plans):
        recv = torch.cat([sends[s][r] for s in range(g)])
        out.append(shard.assemble([recv], [place], int(bounds[r + 1] - bounds[r]), torch.device("cuda")))
    got = torch.cat(out).cpu().numpy().view(np.uint32)
    assert np.array_equal(got, port.reference_index(v).words), (name, g)


@pytest.mark.parametrize("owned", [False, True])
def test_build_distributed_world1_nccl(port, owned):
    """build_distributed end to end through torch.distributed (NCCL, world
    size 1: one process, nothing waits on another rank): the gathered index
    and the owned slice both equal the reference's."""
    import socket

    import torch
    import torch.distributed as dist

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port_num = s.getsockname()[1]
    s.close()
    store = dist.TCPStore("127.0.0.1", port_num, 1, True)
    dist.init_process_group("nccl", store=store, rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        v = gen.zipf(42, 1 << 20, 65536, 1.0)
        sb = shard.ShardBuilder(v.size)
        ent, res = shard.build_distributed(v, 0, sb, owned=owned)
        ref = port.reference_index(v)
        assert np.array_equal(ent, ref.entries)
        if owned:
            bounds, words = res
            assert bounds.tolist() == [0, ref.words.size]
        else:
            words = res
        assert np.array_equal(words.cpu().numpy().view(np.uint32), ref.words)
    finally:
        dist.destroy_process_group()


def _dist_plan_pull(v: np.ndarray, g: int, cap: int = 0):
    """The step's device work (ndx_dist_plan + ndx_dist_pull) over g shards
    built on this GPU: the counts stay on the device, every rank's slice and
    the gathered array are pulled from g separate word buffers (what the
    ranks map over NVLink)."""
    import ctypes

    import torch

    from paper_1709_07781_b200 import ndx

    L = ndx.load()
    sb = shard.ShardBuilder(1 << 16)
    b = shard.shard_bounds(v.size, g).astype(np.int64)
    metas, staged, D = [], [], []
    for k in range(g):
        part = v[b[k]:b[k + 1]]
        if part.size == 0:
            metas.append(np.zeros(0, shard.META_DTYPE))
            staged.append(torch.zeros(1, dtype=torch.int32, device="cuda"))
            D.append(0)
            continue
        keys = torch.from_numpy(part.view(np.int32).copy()).cuda()
        W, d, meta = sb.build(keys, part.size, int(b[k]))
        metas.append(meta[: d * 8].cpu().numpy().view(shard.META_DTYPE).copy())
        staged.append(sb.words[: max(W, 1)].clone())
        D.append(d)
    cap = cap or max(D + [1])
    pad = np.zeros((g, cap), shard.META_DTYPE)
    for k, m in enumerate(metas):
        pad[k, : min(m.size, cap)] = m[:cap]
    counts = np.zeros((g, 3), np.uint64)  # ndx_wah_counts: words, distinct, min | max << 32 (24 B)
    counts[:, 1] = D
    dev = torch.device("cuda")
    d_meta = torch.from_numpy(pad.view(np.int32).copy()).to(dev)
    d_counts = torch.from_numpy(counts.view(np.int32).copy()).to(dev)
    rec = g * cap
    entries = torch.empty(3 * rec + 3, dtype=torch.int32, device=dev)
    merged = torch.empty((rec + 1) * 6, dtype=torch.int32, device=dev)
    totals = torch.zeros(8, dtype=torch.int32, device=dev)
    bounds = torch.zeros(2 * (g + 1), dtype=torch.int32, device=dev)
    scr = torch.empty(L.ndx_dist_plan_scratch_bytes(g, cap) // 4 + 64, dtype=torch.int32, device=dev)
    s = torch.cuda.current_stream().cuda_stream
    P = ndx._ptr
    ndx.check(L.ndx_dist_plan(P(d_meta), cap, P(d_counts), g, P(entries), P(merged), P(totals), P(bounds), P(scr), s),
              "dist_plan")
    tot = totals.cpu().numpy().view(np.uint64)
    Dt, Wt, err = int(tot[0]), int(tot[1]), int(tot[2])
    srcs = (ctypes.c_void_p * g)(*[t.data_ptr() for t in staged])
    out_all = torch.zeros(max(Wt, 1), dtype=torch.int32, device=dev)
    ndx.check(L.ndx_dist_pull(srcs, g, P(merged), rec, P(totals), P(bounds), 0, 1, P(out_all), Wt, Wt, s), "pull")
    bnd = bounds.cpu().numpy().view(np.uint64).astype(np.int64)
    slices = []
    for h in range(g):
        o = torch.zeros(max(int(bnd[h + 1] - bnd[h]), 1), dtype=torch.int32, device=dev)
        ndx.check(L.ndx_dist_pull(srcs, g, P(merged), rec, P(totals), P(bounds), h, 0, P(o), o.numel(), o.numel(),
                                  s), "pull")
        slices.append(o[: int(bnd[h + 1] - bnd[h])])
    err |= int(totals.cpu().numpy().view(np.uint64)[2])
    ent = entries[: 3 * Dt].cpu().numpy().view(np.uint32).reshape(-1, 3)
    return ent, out_all[:Wt].cpu().numpy().view(np.uint32), torch.cat(slices).cpu().numpy().view(np.uint32), bnd, err


@pytest.mark.parametrize("g", [1, 2, 3, 8])
@pytest.mark.parametrize("name", sorted(H.columns()))
def test_device_counts_plan_and_peer_pull(port, name, g):
    """SURVEY 8(e) steps 2-4 as the timed multi-GPU step runs them: plan from
    device counts, then the gathered array and every rank's owned slice
    pulled from the shards' word buffers; both equal the reference index."""
    v = H.columns()[name]
    ent, words, sliced, bnd, err = _dist_plan_pull(v, g)
    ref = port.reference_index(v)
    assert err == 0
    assert np.array_equal(ent, ref.entries) and np.array_equal(words, ref.words), (name, g)
    assert np.array_equal(sliced, ref.words) and bnd[0] == 0 and bnd[-1] == ref.words.size
    assert np.all(np.isin(bnd[1:-1], np.append(ref.entries[:, 1], ref.words.size)))  # cuts at value starts


def test_device_plan_flags_metadata_overflow(port):
    v = gen.uniform(7, 200_000, 5000)
    _, _, _, _, err = _dist_plan_pull(v, 2, cap=1000)
    assert err & 4


@pytest.mark.parametrize("g", [2, 8])
def test_device_plan_zipf_digest(port, g):
    v = gen.zipf(42, 1 << 22, 65536, 1.0)
    ent, words, sliced, _, err = _dist_plan_pull(v, g)
    assert err == 0 and np.array_equal(words, sliced)
    assert port.digest_parts(v.size, ent, words) == port.digest_of(v)


@pytest.mark.parametrize("gather", [False, True])
def test_dist_build_world1_through_runtime(port, gather):
    """The C++ DistBuild (shard chain of compute actors, NCCL all-gather from
    the runtime, device plan, peer pull) at world size 1 -- the code path the
    N > 1 bench times; with a nonzero row base the result is the shifted
    index (the first shard keeps its leading zero-fill)."""
    import torch

    from paper_1709_07781_b200.runtime import DistBuild, Runtime

    rt = Runtime()
    try:
        v = gen.zipf(42, 1 << 20, 65536, 1.0)
        keys = torch.from_numpy(v.view(np.int32).copy()).cuda()
        d = DistBuild(rt, 0, 1, DistBuild.unique_id(), v.size, 1 << 16)
        for base in (0, 31 * 1000):
            d.step(keys.data_ptr(), v.size, base, gather_all=gather)
            rt.synchronize()
            o = d.outputs()
            tot = np.zeros(4, np.uint64)
            from paper_1709_07781_b200 import ndx
            L = ndx.load()
            ndx.check(L.ndx_memcpy_d2h_async(tot.ctypes.data, o["totals"], 32, None), "d2h")
            ndx.check(L.ndx_device_synchronize(), "sync")
            D, W, err = int(tot[0]), int(tot[1]), int(tot[2])
            assert err == 0
            ent = np.zeros(3 * D, np.uint32)
            w = np.zeros(W, np.uint32)
            ndx.check(L.ndx_memcpy_d2h_async(ent.ctypes.data, o["entries"], 12 * D, None), "d2h")
            ndx.check(L.ndx_memcpy_d2h_async(w.ctypes.data, o["slice"], 4 * W, None), "d2h")
            ndx.check(L.ndx_device_synchronize(), "sync")
            ref = port.reference_index(v)
            if base:
                from tests.test_wah_gpu import _shift_index
                want_e, want_w = _shift_index(ref, base // 31)
            else:
                want_e, want_w = ref.entries, ref.words
            assert np.array_equal(ent.reshape(-1, 3), want_e) and np.array_equal(w, want_w), base
        d.close()
    finally:
        rt.close()
