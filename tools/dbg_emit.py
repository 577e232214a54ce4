"""Find and describe the first build that differs from the oracle (GPU)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402
from paper_1709_07781_b200 import gen, ndx  # noqa: E402


def describe(v, got, want):
    print("n", v.size, "D got/want", len(got.entries), len(want.entries), "W", got.words.size, want.words.size)
    for i, (a, b) in enumerate(zip(got.entries.tolist(), want.entries.tolist())):
        if a != b:
            print("first entry diff", i, a, b)
            val = b[0]
            rows = np.nonzero(v == val)[0]
            print(" value", val, "rows", rows.size, "first rows", rows[:40].tolist())
            gw = got.words[a[1]:a[1] + a[2]].tolist()
            ww = want.words[b[1]:b[1] + b[2]].tolist()
            for k, (x, y) in enumerate(zip(gw, ww)):
                if x != y:
                    print(" word", k, hex(x), hex(y), "ctx got", [hex(t) for t in gw[max(0, k - 3):k + 3]],
                          "want", [hex(t) for t in ww[max(0, k - 3):k + 3]])
                    break
            return
    d = np.nonzero(got.words[:min(got.words.size, want.words.size)] != want.words[:min(got.words.size, want.words.size)])[0]
    for k in d[:4]:
        print(" word", k, "got", [hex(t) for t in got.words[max(0, k - 2):k + 3].tolist()], "want", [hex(t) for t in want.words[max(0, k - 2):k + 3].tolist()])
    print(" values first 70:", v[:70].tolist())
    print("entries equal; words differ at", np.nonzero(got.words[:min(got.words.size, want.words.size)] != want.words[:min(got.words.size, want.words.size)])[0][:10])


def main():
    b = ndx.WahBuilder(1 << 20)
    port = oracle.Port()
    inst = gen.instances(20260822, 100, [1, 2, 10, 1000], 100000)
    for i, v in enumerate(inst):
        got = b.build(v)
        want = port.reference_index(v)
        if not (np.array_equal(got.entries, want.entries) and np.array_equal(got.words, want.words)):
            print("instance", i)
            describe(v, got, want)
            break
    rng = np.random.default_rng(1)
    for it in range(300):
        n = int(rng.integers(1, 5000))
        card = int(rng.choice([1, 2, 3, 10]))
        v = rng.integers(0, card, n).astype(np.uint32)
        got = b.build(v)
        want = port.reference_index(v)
        if not (np.array_equal(got.entries, want.entries) and np.array_equal(got.words, want.words)):
            print("random", it, "card", card)
            describe(v, got, want)
            break


if __name__ == "__main__":
    main()
