"""GPU query side against the oracle: decode, encode (CanonicalWriter),
rows_for and AND / OR / AND-NOT of index bitmaps, bit-exact."""
import numpy as np
import pytest

from paper_1709_07781_b200 import gen, query

pytestmark = pytest.mark.gpu


def _bitmaps(rng):
    out = [np.zeros(0, bool), np.ones(31, bool), np.zeros(62, bool), np.ones(100, bool), np.zeros(1, bool)]
    for n in (1, 30, 31, 32, 93, 1000, 31 * 500 + 7):
        for p in (0.0, 0.02, 0.5, 0.98, 1.0):
            out.append(rng.random(n) < p)
        runs = np.repeat(rng.random(max(n // 40, 1)) < 0.5, 40)[:n]
        out.append(runs)
    return out


def test_encode_matches_canonical_writer(port):
    q = query.Query()
    rng = np.random.default_rng(3)
    for b in _bitmaps(rng):
        assert np.array_equal(q.encode(b), port.encode(b.astype(np.uint8))), b.size


def test_decode_matches_reference(port):
    q = query.Query()
    rng = np.random.default_rng(4)
    for b in _bitmaps(rng):
        w = port.encode(b.astype(np.uint8))
        assert np.array_equal(q.decode(w), port.decode(w).astype(bool)), b.size


def test_decode_rejects_zero_length_fill():
    q = query.Query()
    with pytest.raises(ValueError):
        q.decode(np.array([0x1, 0x80000000], np.uint32))


def _device_index(builder, v):
    import torch

    got = builder.build(v)
    d_words = torch.from_numpy(got.words.view(np.int32).copy()).cuda()
    return query.DeviceIndex(v.size, got.entries, d_words)


@pytest.mark.parametrize("card", [1, 3, 50, 1000])
def test_rows_for_matches_reference(builder, port, card):
    v = gen.uniform(17, 100_000, card)
    idx = _device_index(builder, v)
    for value in list(range(min(card, 6))) + [card + 5]:
        assert np.array_equal(idx.rows_for(value), port.rows_for(v, value)), value


@pytest.mark.parametrize("op", ["and", "or", "andnot"])
def test_bitmap_algebra_over_the_index(builder, port, op):
    # clustered + uniform values so fills and literals both occur
    v = np.concatenate([np.repeat(np.arange(40) % 3, 300), gen.uniform(9, 50_000, 4)]).astype(np.uint32)
    idx = _device_index(builder, v)
    for a, b in [(0, 1), (1, 2), (0, 0), (2, 3)]:
        ba, bb = v == a, v == b
        want = {"and": ba & bb, "or": ba | bb, "andnot": ba & ~bb}[op]
        last = np.nonzero(want)[0]
        ref = port.encode(want[: last[-1] + 1].astype(np.uint8)) if last.size else np.zeros(0, np.uint32)
        assert np.array_equal(idx.combine(op, a, b), ref), (op, a, b)


def test_cli_index_file_is_the_reference_index(tmp_path, port):
    """p/tests/test_cli.cpp:61-80: `--seed 5 index build --rows 3000
    --cardinality 7 --verify --output f` writes the reference index byte for
    byte."""
    import oracle
    from paper_1709_07781_b200 import cli

    out = tmp_path / "cli_index.wah"
    assert cli.main(["index", "build", "--seed", "5", "--rows", "3000", "--cardinality", "7", "--verify",
                     "--output", str(out)]) == 0
    v = gen.uniform(5, 3000, 7)
    assert out.read_bytes() == port.reference_index(v).serialize()
    raw = tmp_path / "vals.raw"
    v.astype("<u4").tofile(raw)
    out2 = tmp_path / "from_raw.wah"
    assert cli.main(["index", "build", "--input", str(raw), "--verify", "--output", str(out2)]) == 0
    assert out2.read_bytes() == out.read_bytes()
