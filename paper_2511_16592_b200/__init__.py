"""B200-native GFlowNet training engine (gfnx hot path, arXiv 2511.16592).

The numeric path lives in libgfnx.so (csrc/, sm_100a CUDA behind a C ABI, include/gfnx.h);
``engine.Trainer`` is the host-side mirror of the reference training API.
"""
from . import abi  # noqa: F401
