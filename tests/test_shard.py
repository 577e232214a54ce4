"""Multi-GPU build host logic on CPU: row shards, the merge plan of SURVEY.md
Appendix B (libndactor.so, ndactor_merge_plan) and the torch.distributed
exchange over gloo with world_size 2.  Every merged index must equal the
oracle's index of the whole column, bit for bit."""
import os

import numpy as np
import pytest

from paper_1709_07781_b200 import shard
from tests import shard_helpers as H


@pytest.mark.parametrize("n,g", [(1, 1), (30, 2), (31, 2), (100, 3), (310, 4), (10**6 + 7, 8), (2**30, 8)])
def test_shard_bounds(n, g):
    b = shard.shard_bounds(n, g)
    assert b[0] == 0 and b[-1] == n and np.all(np.diff(b.astype(np.int64)) >= 0)
    assert all(int(x) % 31 == 0 for x in b[:-1])
    sizes = np.diff(b.astype(np.int64))
    if n >= 31 * g:
        assert sizes.max() - sizes.min() <= 31


def _merged(port, v, g):
    b = shard.shard_bounds(v.size, g).astype(np.int64)
    metas, words = [], []
    for k in range(g):
        part = v[b[k]:b[k + 1]]
        if part.size == 0:
            metas.append(np.zeros(0, shard.META_DTYPE))
            words.append(np.zeros(0, np.uint32))
            continue
        e, w = H.local_index(port, part, int(b[k]))
        metas.append(H.local_meta(part, int(b[k]), e, w))
        words.append(w)
    entries, pieces, total = shard.plan_merge(metas)
    return entries, H.assemble(words, pieces, total)


@pytest.mark.parametrize("g", [1, 2, 3, 4, 8])
@pytest.mark.parametrize("name", sorted(H.columns()))
def test_merge_plan_matches_whole_column(port, name, g):
    v = H.columns()[name]
    entries, words = _merged(port, v, g)
    ref = port.reference_index(v)
    assert np.array_equal(entries, ref.entries), (name, g)
    assert np.array_equal(words, ref.words), (name, g)


def test_merge_plan_fuses_ones_over_cuts(port):
    entries, words = _merged(port, np.full(93, 7, np.uint32), 3)
    assert words.tolist() == [0xC0000003] and entries.tolist() == [[7, 0, 1]]


def test_merge_plan_rejects_unsorted():
    m = np.zeros(2, shard.META_DTYPE)
    m["value"] = [5, 3]
    m["body_len"] = 1
    with pytest.raises(Exception):
        shard.plan_merge([m])


def _worker(rank, ws, port_num, q):
    try:
        import torch.distributed as dist
        import torch
        import oracle

        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port_num)
        dist.init_process_group("gloo", rank=rank, world_size=ws)
        port = oracle.Port()
        v = H.columns()["hot_cold"]
        b = shard.shard_bounds(v.size, ws).astype(np.int64)
        part = v[b[rank]:b[rank + 1]]
        e, w = H.local_index(port, part, int(b[rank]))
        metas = shard.exchange_meta(H.local_meta(part, int(b[rank]), e, w))
        entries, pieces, total = shard.plan_merge(metas)
        staged = shard.gather_words(torch.from_numpy(w.view(np.int32).copy()))
        if rank == 0:
            merged = H.assemble([s.numpy().view(np.uint32) for s in staged], pieces, total)
            ref = port.reference_index(v)
            q.put(bool(np.array_equal(merged, ref.words) and np.array_equal(entries, ref.entries)))
        else:
            q.put(bool(len(entries) > 0))
        dist.destroy_process_group()
    except Exception as ex:  # pragma: no cover - reported through the queue
        q.put(repr(ex))


def test_distributed_exchange_gloo_world2():
    import socket
    import torch.multiprocessing as mp

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port_num = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, 2, port_num, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    assert res == [True, True], res


@pytest.mark.parametrize("block", [1, 2, 3, 64])
def test_split_pieces_same_result(port, block):
    v = H.columns()["ones_across"]
    v = np.concatenate([v, H.columns()["hot_cold"]])
    b = shard.shard_bounds(v.size, 3).astype(np.int64)
    metas, words = [], []
    for k in range(3):
        part = v[b[k]:b[k + 1]]
        e, w = H.local_index(port, part, int(b[k]))
        metas.append(H.local_meta(part, int(b[k]), e, w))
        words.append(w)
    entries, pieces, total = shard.plan_merge(metas)
    split = [shard.split_pieces(p, block) for p in pieces]
    assert np.array_equal(H.assemble(words, split, total), H.assemble(words, pieces, total))


def test_merge_plan_padded_input_equals_concatenated(port):
    v = H.columns()["hot_cold"]
    b = shard.shard_bounds(v.size, 4).astype(np.int64)
    metas = []
    for k in range(4):
        part = v[b[k]:b[k + 1]]
        e, w = H.local_index(port, part, int(b[k]))
        metas.append(H.local_meta(part, int(b[k]), e, w))
    cap = max(m.size for m in metas) + 3
    pad = np.zeros((4, cap), shard.META_DTYPE)
    for g, m in enumerate(metas):
        pad[g, :m.size] = m
    e1, p1, w1 = shard.plan_merge(metas)
    e1, p1 = e1.copy(), [p.copy() for p in p1]  # results are views of reused buffers
    e2, p2, w2 = shard.plan_merge(pad, [m.size for m in metas])
    assert w1 == w2 and np.array_equal(e1, e2)
    assert all(np.array_equal(a, b_) for a, b_ in zip(p1, p2))


def test_query_chunk_helpers_round_trip():
    from paper_1709_07781_b200 import query

    rng = np.random.default_rng(1)
    for n in (0, 1, 30, 31, 32, 100, 1000):
        b = rng.random(n) < 0.3
        c = query.bits_to_chunks(b)
        assert c.size == (n + 30) // 31 and (c < (1 << 31)).all()
        assert np.array_equal(query.chunks_to_bits(c, n), b)


def _local_parts(port, v, g):
    b = shard.shard_bounds(v.size, g).astype(np.int64)
    metas, words = [], []
    for k in range(g):
        part = v[b[k]:b[k + 1]]
        if part.size == 0:
            metas.append(np.zeros(0, shard.META_DTYPE))
            words.append(np.zeros(0, np.uint32))
            continue
        e, w = H.local_index(port, part, int(b[k]))
        metas.append(H.local_meta(part, int(b[k]), e, w))
        words.append(w)
    entries, pieces, total = shard.plan_merge(metas)
    return words, entries.copy(), [p.copy() for p in pieces], total


@pytest.mark.parametrize("g", [1, 2, 3, 4, 8])
@pytest.mark.parametrize("name", sorted(H.columns()))
def test_owned_slices_tile_the_whole_index(port, name, g):
    """All-to-all-v by value range, the exchange
    simulated by slicing: every rank's owned slice, concatenated in rank
    order, is the reference index's word array."""
    v = H.columns()[name]
    words, entries, pieces, total = _local_parts(port, v, g)
    bounds = shard.owner_bounds(entries, total, g)
    assert bounds[0] == 0 and bounds[-1] == total and np.all(np.diff(bounds) >= 0)
    assert set(bounds[1:-1].tolist()) <= set(entries[:, 1].tolist()) | {total}  # cuts at value starts
    plans = [shard.owned_plan(pieces, bounds, r) for r in range(g)]
    sends = []
    for r, (pack, sc, place, rc) in enumerate(plans):
        sends.append(np.split(H.assemble([words[r]], [pack], int(sc.sum())), np.cumsum(sc)[:-1]))
    out = []
    for r, (pack, sc, place, rc) in enumerate(plans):
        recv = np.concatenate([sends[s][r] for s in range(g)])
        assert recv.size == int(rc.sum())
        out.append(H.assemble([recv], [place], int(bounds[r + 1] - bounds[r])))
    assert np.array_equal(np.concatenate(out), port.reference_index(v).words), (name, g)


def _owned_worker(rank, ws, port_num, q):
    try:
        import torch
        import torch.distributed as dist
        import oracle

        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port_num)
        dist.init_process_group("gloo", rank=rank, world_size=ws)
        port = oracle.Port()
        v = np.concatenate([H.columns()["hot_cold"], H.columns()["ones_across"]])
        b = shard.shard_bounds(v.size, ws).astype(np.int64)
        part = v[b[rank]:b[rank + 1]]
        e, w = H.local_index(port, part, int(b[rank]))
        metas = shard.exchange_meta(H.local_meta(part, int(b[rank]), e, w))
        entries, pieces, total = shard.plan_merge(metas)
        bounds = shard.owner_bounds(entries, total, ws)
        pack, sc, place, rc = shard.owned_plan(pieces, bounds, rank)
        send = torch.from_numpy(H.assemble([w], [pack], int(sc.sum())).view(np.int32).copy())
        recv = shard.alltoallv_words(send, sc, rc).numpy().view(np.uint32)
        mine = H.assemble([recv], [place], int(bounds[rank + 1] - bounds[rank]))
        ref = port.reference_index(v).words[bounds[rank]:bounds[rank + 1]]
        q.put(bool(np.array_equal(mine, ref) and mine.size > 0))
        dist.destroy_process_group()
    except Exception as ex:  # pragma: no cover - reported through the queue
        q.put(repr(ex))


def test_owned_slices_alltoallv_gloo_world2():
    import socket
    import torch.multiprocessing as mp

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port_num = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_owned_worker, args=(r, 2, port_num, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    assert res == [True, True], res
