"""Generate the golden fixtures FROM THE REFERENCE ITSELF (TEST INFRASTRUCTURE).

Runs the unmodified reference library (oracle/_ref/libndref.so, compiled from
/root/reference by oracle/Makefile) and records:
  small_cases.npz   inputs + expected serialized index bytes (byte-exact)
  digests.json      FNV-1a-64 of serialize_index for generated workloads
                    (generator spec + digest + W + D), incl. the BASELINE
                    configs C1, C3, C4 and the acceptance gate's 100 instances.
Run here (where /root/reference exists):  python tests/golden/make_golden.py
"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402
from paper_1709_07781_b200 import gen  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def small_inputs():
    rng = np.random.default_rng(20261018)
    cases = {
        "hand_5575": np.array([5, 5, 7, 5], np.uint32),                     # test_wah.cpp:133-143
        "solo_100x42": np.full(100, 42, np.uint32),                          # test_wah.cpp:145-149
        "sparse_0_99": np.where(np.isin(np.arange(100), [0, 99]), 9, 1).astype(np.uint32),  # :151-159
        "single_row": np.array([77], np.uint32),                             # test_wah_device.cpp:232-237
        "cli_seed5": gen.uniform(5, 3000, 7),                                # test_cli.cpp:61-80
        "clustered_ones": np.repeat(np.arange(200) % 3, 150).astype(np.uint32),  # test_wah_device.cpp:218-230
        "extremes": np.array([0xFFFFFFFF, 0, 0x80000000, 0xFFFFFFFF, 7, 0x80000000] * 50, np.uint32),
        "all_equal_1000": np.full(1000, 0xDEADBEEF, np.uint32),
        "range_2047": (np.arange(5000) * 7919 % 2048).astype(np.uint32),
        "range_2048": (np.arange(5000) * 7919 % 2049).astype(np.uint32) + 100,
        "full_u32": rng.integers(0, 2**32, 3000, dtype=np.uint64).astype(np.uint32),
        "sorted_runs": np.repeat(np.arange(7, dtype=np.uint32) * 1000003, 620),
        "ones_then_gap": np.concatenate([np.full(93, 4, np.uint32), np.full(31, 5, np.uint32),
                                         np.full(62, 4, np.uint32), np.full(17, 5, np.uint32)]),
    }
    for i, card in enumerate([1, 2, 10, 1000]):
        n = int(rng.integers(1, 3000))
        cases[f"rand_card{card}"] = (rng.integers(0, card, n).astype(np.uint32) * 37 + 11)
    return cases


def main():
    ref = oracle.Reference()
    small = small_inputs()
    npz = {}
    for name, v in small.items():
        idx = ref.reference_index(v)
        npz[f"in_{name}"] = v
        npz[f"out_{name}"] = np.frombuffer(idx.serialize(), np.uint8)
    np.savez_compressed(os.path.join(HERE, "small_cases.npz"), **npz)
    print("small cases:", len(small))

    digests = {"generator": "libstdc++ (g++ 13.3) distributions; see paper_1709_07781_b200/gen.py",
               "workloads": [], "acceptance": None}

    def add(spec, values):
        t = time.time()
        idx = ref.reference_index(values)
        d = dict(spec, digest="%016x" % idx.digest(), W=int(idx.words.size), D=int(len(idx.entries)),
                 ref_seconds=round(time.time() - t, 2))
        digests["workloads"].append(d)
        print(d, flush=True)

    for n, k in [(1 << 20, 256), (1 << 22, 1024), (1 << 24, 256), (1 << 26, 1024), (1 << 26, 65536)]:
        add(dict(kind="uniform", seed=1, n=n, k=k), gen.uniform(1, n, k))
    for n in [1 << 20, 1 << 24, 1 << 28]:
        add(dict(kind="zipf", seed=42, n=n, k=65536, s=1.0), gen.zipf(42, n, 65536, 1.0))

    inst = gen.instances(20260822, 100, [1, 2, 10, 1000], 100000)  # acceptance.cpp:56-79
    digests["acceptance"] = dict(seed=20260822, count=100, cards=[1, 2, 10, 1000], max_rows=100000,
                                 digests=["%016x" % ref.digest_of(v) for v in inst])
    with open(os.path.join(HERE, "digests.json"), "w") as f:
        json.dump(digests, f, indent=1)
    print("wrote digests.json")


if __name__ == "__main__":
    main()
