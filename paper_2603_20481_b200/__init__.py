"""specsense-b200: B200-native (sm_100a) spectrum-occupancy detection hot path.

The reference (arXiv 2603.20481, "RISE") is a C++20 library; this package
holds the CUDA kernels + C ABI + C++ drop-in (csrc/, built in-tree into
_lib/libspecsense_b200.so) and a Python mirror of the reference's stage API
(specsense.py) used by the tests and bench.py.
"""
from . import _native  # noqa: F401

__all__ = ["_native", "specsense", "signals"]
