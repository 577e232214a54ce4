"""Build libndx variants (NDX_DEFINES) as lib/libndx_<name>.so for timing
experiments, e.g.
    python tools/variants.py v1=-DNDX_EXP_NOLOOKBACK v2="-DNDX_SORT_MINB=2"
then on the GPU:  NDX_LIB=libndx_v1.so python tools/stage_times.py C4
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1709_07781_b200 import _build  # noqa: E402

for arg in sys.argv[1:]:
    name, _, defs = arg.partition("=")
    os.environ["NDX_OUT"] = f"libndx_{name}.so"
    os.environ["NDX_DEFINES"] = defs
    _build.build_ndx(force=True)
