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
