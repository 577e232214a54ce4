"""The C++ runtime's contract tests (tests/cpp, restating the reference's
test_actor / test_device / test_compute / test_wah_device / test_wah suites)
and the runtime's C ABI from Python."""
import os
import subprocess

import numpy as np
import pytest

from paper_1709_07781_b200 import _build

BIN = os.path.join(_build.LIB, "ndactor_tests")


def _run(group):
    if not os.path.exists(BIN):
        _build.build_all()
    p = subprocess.run([BIN, group], capture_output=True, text=True, timeout=900)
    tail = "\n".join(p.stdout.splitlines()[-40:])
    assert p.returncode == 0, tail + p.stderr[-2000:]
    return p.stdout


def test_cpp_cpu_contract():
    out = _run("cpu")
    assert "0 failed" in out


@pytest.mark.gpu
def test_cpp_gpu_contract():
    out = _run("gpu")
    assert "0 failed" in out


@pytest.mark.gpu
def test_runtime_c_abi_build_index_matches_oracle(port):
    from paper_1709_07781_b200 import gen
    from paper_1709_07781_b200.runtime import Runtime

    rt = Runtime()
    for v in [gen.uniform(5, 3000, 7), gen.zipf(42, 1 << 20, 65536), np.zeros(0, np.uint32),
              np.repeat(np.arange(9, dtype=np.uint32), 10_000)]:
        n, ent, words = rt.build_index(v)
        want = port.reference_index(v)
        assert np.array_equal(words, want.words) and np.array_equal(ent, want.entries)
    rt.close()


@pytest.mark.gpu
def test_runtime_dispatch_probe_counts_every_kernel():
    from paper_1709_07781_b200.runtime import Runtime

    rt = Runtime()
    raw_ms, actor_ms, check = rt.dispatch_probe(2000)
    assert check == 4000
    assert raw_ms > 0 and actor_ms > 0
    rt.close()


@pytest.mark.gpu
def test_runtime_async_pipeline_matches_oracle(port):
    """ndactor_wah_build_index_async: two builds in flight, results copied
    to pinned host memory on the egress stream, bit-exact."""
    import torch

    from paper_1709_07781_b200 import gen
    from paper_1709_07781_b200.runtime import Runtime

    rt = Runtime()
    cols = [gen.uniform(11, 300_000, 1000), gen.zipf(5, 500_000, 4096, 1.0), gen.uniform(12, 77_777, 3),
            np.full(40_000, 9, np.uint32)]
    pin = lambda k: torch.empty(k, dtype=torch.int32, pin_memory=True).numpy().view(np.uint32)  # noqa: E731
    ins = [pin(v.size) for v in cols]
    for a, v in zip(ins, cols):
        a[:] = v
    outs = [(pin(2 * v.size), pin(3 * 4096 + 64), torch.zeros(3, dtype=torch.int64, pin_memory=True).numpy().view(np.uint64))
            for v in cols]
    pending = []
    for i, v in enumerate(cols):
        if len(pending) == 2:
            j, t = pending.pop(0)
            rt.wait(t)
        pending.append((i, rt.build_index_async(ins[i], *outs[i])))
    for _, t in pending:
        rt.wait(t)
    for v, (w, e, c) in zip(cols, outs):
        ref = port.reference_index(v)
        W, D = int(c[0]), int(c[1])
        assert W == ref.words.size and D == len(ref.entries)
        assert np.array_equal(w[:W], ref.words) and np.array_equal(e[:3 * D].reshape(-1, 3), ref.entries)
    rt.close()


@pytest.mark.gpu
def test_runtime_async_small_capacity_and_pageable(port):
    """Capacities below the result: the true counts come back and exactly
    the prefix that fits is written (nothing past it); pageable output
    memory works too."""
    from paper_1709_07781_b200 import gen
    from paper_1709_07781_b200.runtime import Runtime

    rt = Runtime()
    v = gen.zipf(9, 200_000, 2000, 1.0)
    ref = port.reference_index(v)
    W, D = ref.words.size, len(ref.entries)
    w = np.full(W // 3 + 2, 0xDEADBEEF, np.uint32)
    e = np.full(3 * (D // 2) + 3, 0xDEADBEEF, np.uint32)
    c = np.zeros(3, np.uint64)
    rt.wait(rt.build_index_async(v, w[:-2], e[:-3], c))
    assert int(c[0]) == W and int(c[1]) == D
    assert np.array_equal(w[:-2], ref.words[:w.size - 2]) and (w[-2:] == 0xDEADBEEF).all()
    assert np.array_equal(e[:-3], ref.entries.reshape(-1)[:e.size - 3]) and (e[-3:] == 0xDEADBEEF).all()
    # zero capacities: counts only
    c2 = np.zeros(3, np.uint64)
    rt.wait(rt.build_index_async(v, w[:0], e[:0], c2))
    assert int(c2[0]) == W and int(c2[1]) == D
    rt.close()
