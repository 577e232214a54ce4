"""In-tree build of the native libraries (no JIT cache: the .so files travel
with the repo snapshot to the GPU box).

  lib/libndx.so      CUDA kernels + device C ABI (include/ndx.h), sm_100a
  lib/libndactor.so  C++ host runtime: actors, MemRef, compute actors, WAH API
                     (include/ndactor/*.hpp) + its C ABI (include/ndactor_c.h)
  lib/ndactor_tests  C++ contract tests of the runtime (tests/cpp/*.cpp)
"""
from __future__ import annotations

import glob
import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
LIB = os.path.join(PKG, "lib")
CSRC = os.path.join(PKG, "csrc")
INC = os.path.join(ROOT, "include")

NVCC = os.environ.get("NVCC", shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
CUDA_HOME = os.environ.get("CUDA_HOME", "/usr/local/cuda")


def _run(cmd: list[str]) -> None:
    print("+", " ".join(cmd), flush=True)
    subprocess.run(cmd, check=True)


def _stale(out: str, srcs: list[str]) -> bool:
    if not os.path.exists(out):
        return True
    t = os.path.getmtime(out)
    return any(os.path.getmtime(s) > t for s in srcs)


def build_ndx(force: bool = False) -> str:
    # NDX_OUT / NDX_DEFINES build experiment variants next to libndx.so
    # (selected at load time with NDX_LIB); the product is always libndx.so.
    out = os.path.join(LIB, os.environ.get("NDX_OUT", "libndx.so"))
    defines = os.environ.get("NDX_DEFINES", "").split()
    srcs = sorted(glob.glob(os.path.join(CSRC, "kernels", "*.cu")))
    deps = srcs + glob.glob(os.path.join(CSRC, "kernels", "*.cuh")) + [os.path.join(INC, "ndx.h")]
    if force or _stale(out, deps):
        os.makedirs(LIB, exist_ok=True)
        # -rdc: the plan and sort stages launch exactly the kernels the
        # device-made plan needs from the device (tail launches, CDP)
        _run([NVCC, *ARCH, "-O3", "-lineinfo", "-std=c++17", "-rdc=true", "-Xcompiler", "-fPIC,-O3",
              "-Xptxas", "-v" if os.environ.get("NDX_PTXAS_V") else "-O3",
              "--expt-relaxed-constexpr", "-cudart", "static", "-shared", "-I" + INC, *defines,
              "-o", out, *srcs, "-lcudadevrt"])
    return out


def build_ndactor(force: bool = False) -> str:
    out = os.path.join(LIB, "libndactor.so")
    srcs = sorted(glob.glob(os.path.join(CSRC, "runtime", "*.cpp")))
    if not srcs:
        return out
    deps = srcs + glob.glob(os.path.join(CSRC, "runtime", "*.hpp")) + \
        glob.glob(os.path.join(INC, "ndactor", "*.hpp")) + glob.glob(os.path.join(INC, "*.h"))
    if force or _stale(out, deps + [os.path.join(LIB, "libndx.so")]):
        cxx = os.environ.get("CXX", "g++")
        _run([cxx, "-std=c++20", "-O2", "-g", "-fPIC", "-shared", "-pthread", "-I" + INC,
              "-o", out, *srcs, "-L" + LIB, "-lndx", "-ldl", "-Wl,-rpath,$ORIGIN"])
    return out


def build_verify(force: bool = False) -> str:
    """libndactor_verify.so: wah::reference_index for the reference's own
    consumers (ndcli --verify, the acceptance gate).  Not part of the product
    library: nothing in libndactor/libndx links it."""
    out = os.path.join(LIB, "libndactor_verify.so")
    srcs = sorted(glob.glob(os.path.join(CSRC, "verify", "*.cpp")))
    deps = srcs + [os.path.join(INC, "ndactor", "wah.hpp"), os.path.join(LIB, "libndactor.so")]
    if force or _stale(out, deps):
        cxx = os.environ.get("CXX", "g++")
        _run([cxx, "-std=c++20", "-O2", "-fPIC", "-shared", "-I" + INC, "-o", out, *srcs,
              "-L" + LIB, "-lndactor", "-Wl,-rpath,$ORIGIN"])
    return out


def build_cpp_tests(force: bool = False) -> str | None:
    """C++ contract tests (tests/cpp): CPU cases need no GPU; GPU cases use
    real CUDA test kernels and check results against the oracle library."""
    srcs = sorted(glob.glob(os.path.join(ROOT, "tests", "cpp", "*.cpp")) +
                  glob.glob(os.path.join(ROOT, "tests", "cpp", "*.cu")))
    if not srcs:
        return None
    out = os.path.join(LIB, "ndactor_tests")
    oracle_dir = os.path.join(ROOT, "oracle", "_build")
    if not os.path.exists(os.path.join(oracle_dir, "libwah_oracle.so")):
        subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle"), os.path.join("_build", "libwah_oracle.so")],
                       check=True)
    deps = srcs + glob.glob(os.path.join(ROOT, "tests", "cpp", "*.hpp")) + [os.path.join(LIB, "libndactor.so"),
                                                                            os.path.join(LIB, "libndactor_verify.so")]
    if force or _stale(out, deps):
        _run([NVCC, *ARCH, "-O1", "-g", "-std=c++20", "-Xcompiler", "-pthread", "-I" + INC,
              "-o", out, *srcs, "-L" + LIB, "-lndactor_verify", "-lndactor", "-lndx", "-L" + oracle_dir,
              "-lwah_oracle",
              "-Xlinker", "-rpath," + LIB + ":" + oracle_dir, "-cudart", "static"])
    return out


def build_all(force: bool = False) -> None:
    build_ndx(force)
    build_ndactor(force)
    build_verify(force)
    build_cpp_tests(force)


if __name__ == "__main__":
    build_all(force="--force" in sys.argv)
