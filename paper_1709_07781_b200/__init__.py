"""paper_1709_07781_b200 -- B200-native WAH bitmap-index build behind the
reference's actor-facing API (arXiv 1709.07781, "OpenCL Actors").

Native pieces (built in-tree by ``_build.py``):
  lib/libndx.so      sm_100a kernels + device C ABI      (include/ndx.h)
  lib/libndactor.so  C++ host runtime: ActorSystem, MemRef, compute actors,
                     wah::build_index & co.               (include/ndactor/*.hpp,
                                                           include/ndactor_c.h)
Python modules are thin ctypes bindings used by tests and bench.py.
"""
__all__ = ["ndx", "gen", "runtime"]
