"""Test-side helpers for the multi-GPU merge: local shard indexes from the
oracle (shifted to global row ids), their metadata, and a reference
assembly of a merge plan.  Test infrastructure only."""
import numpy as np

from paper_1709_07781_b200.shard import META_DTYPE


def local_index(port, values: np.ndarray, row_base: int):
    """The index a shard build with row_base (a multiple of 31) produces:
    the oracle's index of the shard's values with every value's leading
    zero-fill grown by row_base/31 chunks."""
    k = row_base // 31
    ref = port.reference_index(values)
    out, ents, off = [], [], 0
    for v, o, ln in ref.entries.tolist():
        w = ref.words[o:o + ln].tolist()
        if k:
            if (w[0] & 0xC0000000) == 0x80000000:
                w[0] = 0x80000000 | ((w[0] & 0x3FFFFFFF) + k)
            else:
                w.insert(0, 0x80000000 | k)
        ents.append([v, off, len(w)])
        out += w
        off += len(w)
    return np.array(ents, np.uint32).reshape(-1, 3), np.array(out, np.uint32)


def local_meta(values: np.ndarray, row_base: int, entries: np.ndarray, words: np.ndarray) -> np.ndarray:
    m = np.zeros(len(entries), META_DTYPE)
    for d, (v, off, ln) in enumerate(entries.tolist()):
        rows = np.nonzero(values == v)[0] + row_base
        skip = 1 if (int(words[off]) & 0xC0000000) == 0x80000000 else 0
        first, last = int(words[off + skip]), int(words[off + ln - 1])
        m[d] = (v, rows[0] // 31, rows[-1] // 31,
                first & 0x3FFFFFFF if (first & 0xC0000000) == 0xC0000000 else 0,
                last & 0x3FFFFFFF if (last & 0xC0000000) == 0xC0000000 else 0,
                off + skip, ln - skip, skip)
    return m


def assemble(words_per_shard, pieces, total: int) -> np.ndarray:
    out = np.zeros(total, np.uint32)
    filled = np.zeros(total, bool)
    for w, ps in zip(words_per_shard, pieces):
        for p in ps:
            dst = int(p["dst"])
            if p["lead"]:
                out[dst] = p["lead"]
                filled[dst] = True
                dst += 1
            s, k = int(p["src_off"]), int(p["src_len"])
            out[dst:dst + k] = w[s:s + k]
            filled[dst:dst + k] = True
    assert filled.all(), "plan left holes"
    return out


def columns():
    """Columns that exercise every merge rule."""
    rng = np.random.default_rng(77)
    cols = {
        "ones_across": np.full(310, 7, np.uint32),                  # one stretch over the cut
        "ones_tiny_shards": np.full(93, 7, np.uint32),              # fused over 3 one-chunk shards
        "mixed": rng.integers(0, 40, 20_000).astype(np.uint32),
        "hot_cold": np.where(rng.random(30_000) < 0.9, 3, rng.integers(0, 5000, 30_000)).astype(np.uint32),
        "blocks": np.repeat(np.arange(60) % 4, 217).astype(np.uint32),  # runs of 7 chunks
        "one_shard_values": np.concatenate([np.full(5000, 1), np.full(5000, 2)]).astype(np.uint32),
        "partial_tail": np.concatenate([np.full(31 * 6, 9), np.array([9, 1, 9])]).astype(np.uint32),
        "alternating": (np.arange(4000) % 2).astype(np.uint32),
    }
    return cols
