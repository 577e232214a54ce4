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
