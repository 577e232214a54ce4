"""GPU parity: the sm_100a build (through the C ABI, include/ndx.h) against the
oracle and the reference-generated golden fixtures.  Bit-exact, no tolerance.

Mirrors p/tests/test_wah_device.cpp:45-274 and acceptance.cpp checks 1-3."""
import json
import os
import zlib

import numpy as np
import pytest

from paper_1709_07781_b200 import gen

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden")


def same(got, want):
    return got.row_count == want.row_count and np.array_equal(got.entries, want.entries) and \
        np.array_equal(got.words, want.words)


def test_small_golden_cases(builder, port):
    z = np.load(os.path.join(GOLD, "small_cases.npz"))
    for k in z.files:
        if not k.startswith("in_"):
            continue
        name = k[3:]
        v = z[k]
        got = builder.build(v)
        import oracle

        ser = oracle.Index(got.row_count, got.entries, got.words).serialize()
        assert ser == z["out_" + name].tobytes(), name


def test_random_instances_across_cardinalities(builder, port):  # test_wah_device.cpp:202-216
    rng = np.random.default_rng(8005)
    for it in range(24):
        n = int(rng.integers(1, 30001))
        card = [1, 2, 10, 1000][it % 4]
        v = (rng.integers(0, card, n).astype(np.uint32) * 37 + 11)
        assert same(builder.build(v), port.reference_index(v)), (it, n, card)


def test_clustered_rows_produce_ones_fills(builder, port):  # test_wah_device.cpp:218-230
    v = np.repeat(np.arange(200) % 3, 150).astype(np.uint32)
    got = builder.build(v)
    assert same(got, port.reference_index(v))
    assert any((w & 0xC0000000) == 0xC0000000 for w in got.words.tolist())


def test_single_row_and_empty(builder, port):  # test_wah_device.cpp:232-244
    got = builder.build(np.array([77], np.uint32))
    assert got.words.tolist() == [1] and got.entries.tolist() == [[77, 0, 1]]
    e = builder.build(np.zeros(0, np.uint32))
    assert e.row_count == 0 and e.entries.size == 0 and e.words.size == 0


@pytest.mark.parametrize("case", ["long_stretch", "stretch_tile_edges", "sorted_blocks", "mode_edges",
                                  "full_range", "hi_bytes", "constant", "two_values_alt", "wide_high_base",
                                  "bytes_0_and_2", "wide_high_base_big"])
def test_adversarial_shapes(builder, port, case):
    rng = np.random.default_rng(zlib.crc32(case.encode()))
    if case == "long_stretch":  # ones-stretches spanning many emit tiles
        v = np.repeat(np.array([3, 1, 4, 1, 5], np.uint32), [200_000, 31 * 5000, 93, 31 * 777 + 5, 10])
    elif case == "stretch_tile_edges":
        parts = []
        for L in [31 * 132 - 1, 31 * 132, 31 * 132 + 1, 4096, 4095, 8192 + 31, 62, 30, 31]:
            parts.append(np.full(L, len(parts) % 4, np.uint32))
        v = np.concatenate(parts * 20)
    elif case == "sorted_blocks":
        v = np.sort(rng.integers(0, 5000, 300_000)).astype(np.uint32)
    elif case == "mode_edges":  # key range 2047 / 2048 / 2049 (wide vs byte passes)
        v = np.concatenate([rng.integers(10, 10 + r, 40_000) for r in (2047, 2048, 2049)]).astype(np.uint32)
    elif case == "full_range":  # all four byte passes
        v = rng.integers(0, 2**32, 200_000, dtype=np.uint64).astype(np.uint32)
        v[3] = 0xFFFFFFFF
        v[100] = 0x80000000
    elif case == "hi_bytes":  # bytes 2/3 vary, 0/1 constant
        v = (rng.integers(0, 300, 100_000).astype(np.uint32) << 16) | 0x1234
    elif case == "wide_high_base":  # one wide pass, keys above 2^16 (no narrow packing)
        v = (3_000_000_000 + rng.integers(0, 2000, 150_000)).astype(np.uint32)
    elif case == "wide_high_base_big":  # the same over many full 16384-pair tiles
        v = (0xFFFFF000 + rng.zipf(1.3, 1_500_000) % 2040).astype(np.uint32)
    elif case == "bytes_0_and_2":  # two byte passes with a constant byte between them
        v = (rng.integers(0, 256, 120_000).astype(np.uint32) << 16) | rng.integers(0, 256, 120_000).astype(np.uint32) | 0x4200
    elif case == "constant":
        v = np.full(123_457, 0xFFFFFFFF, np.uint32)
    else:
        v = np.tile(np.array([0xAAAA, 0x5555], np.uint32), 70_001)
    got = builder.build(v)
    want = port.reference_index(v)
    assert same(got, want), case


def _digests():
    with open(os.path.join(GOLD, "digests.json")) as f:
        return json.load(f)


def test_acceptance_instances(builder, port):  # acceptance.cpp:56-79 (check 1)
    a = _digests()["acceptance"]
    inst = gen.instances(a["seed"], a["count"], a["cards"], a["max_rows"])
    for i, (v, d) in enumerate(zip(inst, a["digests"])):
        got = builder.build(v)
        assert "%016x" % port.digest_parts(got.row_count, got.entries, got.words) == d, i


@pytest.mark.parametrize("w", _digests()["workloads"], ids=lambda w: f"{w['kind']}-n{w['n']}-k{w['k']}")
def test_baseline_workload_digests(builder, port, w):
    """C1, C3, C4 and friends: digest of serialize_index equals the reference's."""
    v = gen.uniform(w["seed"], w["n"], w["k"]) if w["kind"] == "uniform" else gen.zipf(w["seed"], w["n"], w["k"], w["s"])
    got = builder.build(v)
    assert got.words.size == w["W"] and len(got.entries) == w["D"]
    assert "%016x" % port.digest_parts(got.row_count, got.entries, got.words) == w["digest"]


@pytest.mark.parametrize("case", ["compact_high_base", "compact_small_many_groups", "compact_segments",
                                  "compact_sparse_across_segments", "compact_one_low_byte_bucket"])
def test_compact_two_pass_mode(builder, port, case):
    """The compact mode (key range >= 2^11, bytes 2/3 constant, 0/1 varying):
    pass A's packed u32 carries the row's low 24 bits; pass B recovers the
    low byte and the row segment from the group tables."""
    rng = np.random.default_rng(zlib.crc32(case.encode()))
    if case == "compact_high_base":  # a nonzero constant top half
        v = (0x12340000 + rng.integers(0, 65536, 300_000)).astype(np.uint32)
    elif case == "compact_small_many_groups":  # more groups than fit a tile's fast path
        v = rng.integers(0, 60_000, 5000).astype(np.uint32)
    elif case == "compact_segments":  # several 2^24-row segments
        v = rng.integers(0, 65536, (1 << 24) * 2 + 12345).astype(np.uint32)
    elif case == "compact_sparse_across_segments":  # a key seen once per distant segment
        v = rng.integers(0, 60_000, (1 << 25) + 100).astype(np.uint32)
        v[5] = 65535
        v[(1 << 25) + 3] = 65535
        v[(1 << 24) + 7] = 65279  # same low byte, another high byte
    else:  # every key shares its low byte: one pass-A bucket
        v = (rng.integers(0, 256, 200_000).astype(np.uint32) << 8) | 0x77
    got = builder.build(v)
    assert same(got, port.reference_index(v)), case


def test_repeat_builds_are_deterministic(builder, port):
    v = gen.uniform(3, 500_000, 300)
    a = builder.build(v)
    for _ in range(3):
        assert same(builder.build(v), a)
    assert same(a, port.reference_index(v))


# ---- device primitives behind the reference's public API -----------------

@pytest.mark.parametrize("n", [1, 2, 1023, 1024, 1025, 4096, 50000, 1048577])
def test_scan_matches_serial_oracle(prims, port, n):  # test_wah_device.cpp:45-61
    x = np.random.default_rng(n).integers(0, 10, n).astype(np.uint32)
    assert np.array_equal(prims.scan_exclusive(x), port.scan_exclusive(x))


def test_scan_wraps_mod_2_32(prims, port):
    x = np.full(100_000, 0xFFFFFFF0, np.uint32)
    assert np.array_equal(prims.scan_exclusive(x), port.scan_exclusive(x))


@pytest.mark.parametrize("n", [1, 7, 16384, 16385, 40000])
def test_sort_pairs_stable(prims, port, n):  # test_wah_device.cpp:63-107
    rng = np.random.default_rng(8002 + n)
    keys = rng.integers(0, 6, n).astype(np.uint32)
    if n > 20:
        keys[3] = 0xFFFFFFFF
        keys[n // 2] = 0x80000000
    pos = np.arange(n, dtype=np.uint32)
    k, p = prims.sort_pairs(keys, pos)
    ek, ep = port.sort_pairs(keys, pos)
    assert np.array_equal(k, ek) and np.array_equal(p, ep)


def test_compaction_drops_zeros_keeps_order(prims, port):  # test_wah_device.cpp:109-133, acceptance 3
    rng = np.random.default_rng(8003)
    for it in range(60):
        n = int(rng.integers(1, 20001))
        if it % 10 == 8:
            x = np.zeros(n, np.uint32)
        elif it % 10 == 9:
            x = rng.integers(1, 100, n).astype(np.uint32)
        else:
            x = rng.integers(0, 3, n).astype(np.uint32)
        assert np.array_equal(prims.compact(x), port.filter_nonzero(x)), it


def _shift_index(ref, k_chunks: int):
    """The index of the same values placed at rows 31*k_chunks + i: every
    value's leading zero-fill grows by k_chunks chunks (Appendix B's shard
    pieces before the merge)."""
    out, ents, off = [], [], 0
    for v, o, ln in ref.entries.tolist():
        w = ref.words[o:o + ln].tolist()
        if (w[0] & 0xC0000000) == 0x80000000:
            w[0] = 0x80000000 | ((w[0] & 0x3FFFFFFF) + k_chunks)
        else:
            w.insert(0, 0x80000000 | k_chunks)
        ents.append([v, off, len(w)])
        out += w
        off += len(w)
    return np.array(ents, np.uint32).reshape(-1, 3), np.array(out, np.uint32)


@pytest.mark.parametrize("k_chunks", [1, 1000, 70_000_000, 100_000_000, 138_000_000])
def test_row_base_shards(builder, port, k_chunks):
    """Shard builds with global row ids (row_base = 31k): the emit stage's
    fast chunk division covers rows < 0x8D3DCB08, larger bases take the
    exact path; both must match the shifted oracle index."""
    rng = np.random.default_rng(k_chunks)
    v = np.concatenate([rng.integers(0, 50, 40_000), np.full(3100, 7), rng.integers(0, 3, 9000)]).astype(np.uint32)
    got = builder.build(v, row_base=31 * k_chunks)
    ents, words = _shift_index(port.reference_index(v), k_chunks)
    assert np.array_equal(got.entries, ents) and np.array_equal(got.words, words)


def _column_from_counts(keys, counts, rng, shuffle=True):
    """A column whose sorted stream has key keys[i] over counts[i] positions
    (value starts at the prefix sums), rows in random order unless not
    shuffled (then each key's rows are one contiguous range)."""
    v = np.repeat(np.asarray(keys, dtype=np.uint32), counts)
    if shuffle:
        rng.shuffle(v)
    return v


@pytest.mark.parametrize("mode", ["wide", "compact"])
@pytest.mark.parametrize("case", ["starts_at_buffer_edges", "heads_per_tile_sweep", "stretch_meets_next_value",
                                  "stretch_after_value_start"])
def test_rows_form_edges(builder, port, mode, case):
    """The rows form (wah_emit.cu k_emit_rows): value starts on and around the
    emit tiles' buffer edges (tile 3584, halo 32 before and 4 after), tiles
    holding about kRecHeads = 60 heads (the record's inline list against the
    walk over vs), and all-ones stretches that end exactly where the next
    value's rows continue the row sequence (the stretch is bounded by the
    value's extent, not by the rows)."""
    rng = np.random.default_rng(zlib.crc32((mode + case).encode()))
    base = 11 if mode == "wide" else 0x00050000
    T = 3584

    def keys(m):  # wide: consecutive keys; compact: spread over both low bytes, top half constant
        return base + (1 if mode == "wide" else max(1, 65535 // m)) * np.arange(m)

    if case == "starts_at_buffer_edges":
        starts = sorted({0, 1, 31, 32, 33} | {t * T + d for t in range(1, 6) for d in (-33, -32, -31, -1, 0, 1, 3, 4, 5)})
        n = 6 * T + 50
        counts = np.diff(starts + [n])
        v = _column_from_counts(keys(len(counts)), counts, rng)
    elif case == "heads_per_tile_sweep":
        counts = []
        for c in range(52, 70):  # 3620 / c heads per buffer: 69 .. 52
            counts += [c] * (2 * T // c)
        counts = np.array(counts)
        v = _column_from_counts(keys(len(counts)), counts, rng)
    elif case == "stretch_meets_next_value":
        # key i holds rows [r_i, r_{i+1}): every value is an all-ones stretch
        # and the next value's first row is this value's last + 1
        counts = rng.integers(20, 200, 300)
        v = _column_from_counts(keys(len(counts)), counts, rng, shuffle=False)
    else:
        # long stretches that start right after another value's start, inside
        # one emit tile and across tiles
        counts = np.array([1, 61, 62, 93, 1, 31, 4000, 2, 7300, 30, 31, 32, 62, 93, 124] * 8)
        v = _column_from_counts(keys(len(counts)), counts, rng, shuffle=False)
    if mode == "wide":
        assert int(v.max()) - int(v.min()) < 2048 or case == "heads_per_tile_sweep"
    assert same(builder.build(v), port.reference_index(v)), (mode, case)


@pytest.mark.parametrize("n", [2047, 2048, 2049, 2048 * 3 + 31, 8191, 8192, 8193, 16383, 16384, 16385,
                               16384 * 3 + 1, 4096 * 37])
@pytest.mark.parametrize("kind", ["uniform", "clustered", "zipf"])
def test_tile_boundaries(builder, port, n, kind):
    """Sizes around the emit tile (2048 pairs), the byte-pass tile (8192)
    and the wide-pass tile (16384), with short and long runs."""
    rng = np.random.default_rng(n)
    if kind == "uniform":
        v = rng.integers(0, 3000, n).astype(np.uint32)
    elif kind == "clustered":
        v = np.repeat(rng.integers(0, 5, (n + 99) // 100), 100)[:n].astype(np.uint32)
    else:
        v = gen.zipf(n, n, 70000, 1.0)
    assert same(builder.build(v), port.reference_index(v)), (n, kind)


@pytest.mark.parametrize("w", _digests().get("gpu_workloads", []), ids=lambda w: f"{w['kind']}-n{w['n']}-k{w['k']}")
def test_largest_workload_digest(w):
    """C5 (2^30 values, 65536 keys) on one GPU: the digest of the index equals
    the oracle's, computed once on the GPU box (74 s of CPU) and stored."""
    import oracle
    from paper_1709_07781_b200 import ndx

    v = gen.uniform(w["seed"], w["n"], w["k"])
    b = ndx.WahBuilder(w["n"])
    got = b.build(v)
    assert got.words.size == w["W"] and len(got.entries) == w["D"]
    assert "%016x" % oracle.Port().digest_parts(got.row_count, got.entries, got.words) == w["digest"]


@pytest.mark.gpu
def test_epoch_wrap_clears_stale_statuses(port):
    """The look-back tags are 24 bits and come round after 2^21 builds.  A
    build that wraps must not be able to read statuses left by the build one
    cycle earlier at tiles no build has reached since: the wrapping build
    clears every status below the buffer's high-water mark."""
    from paper_1709_07781_b200 import ndx

    n = 1 << 21
    b = ndx.WahBuilder(n)
    L = b.lib
    first = gen.zipf(3, n, 65536, 1.0)
    assert same(b.build(first), port.reference_index(first))
    assert int(b.status[0].item()) == 8  # the first build's epoch
    hi = L.ndx_wah_status_bytes(n) // 4
    assert int(b.status[64:hi].count_nonzero().item()) > 0  # statuses of many tiles
    b.status[0] = 0xFFFFF8               # the last epoch of the cycle
    small = gen.zipf(4, 5000, 65536, 1.0)
    assert same(b.build(small), port.reference_index(small))
    assert int(b.status[0].item()) == 8  # wrapped: the first build's tags again
    lo = L.ndx_wah_status_bytes(small.size) // 4
    assert int(b.status[lo:hi].count_nonzero().item()) == 0  # no stale status left
    second = gen.zipf(5, n, 65536, 1.0)
    assert same(b.build(second), port.reference_index(second))
