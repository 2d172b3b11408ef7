"""GPU: tcgen05.mma with the A operand in tensor memory (the rollout's hidden/head GEMM form)
against a float64 product of the same bf16 operands."""
import ctypes as C

import numpy as np
import pytest

from paper_2511_16592_b200 import engine

pytestmark = pytest.mark.gpu


def _bf16(x):
    u = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32)
    r = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16).astype(np.uint16)
    return r, (r.astype(np.uint32) << 16).view(np.float32)


def test_ts_mma_matches_fp64_product():
    rng = np.random.default_rng(0)
    a16, a = _bf16(rng.standard_normal((128, 256)))
    b16, b = _bf16(rng.standard_normal((256, 256)))
    d = np.zeros((128, 256), np.float32)
    L = engine.lib()
    rc = L.gfnx_test_ts_mma(a16.ctypes.data_as(C.c_void_p), b16.ctypes.data_as(C.c_void_p),
                            d.ctypes.data_as(C.c_void_p))
    assert rc == 0
    ref = a.astype(np.float64) @ b.astype(np.float64).T
    assert np.max(np.abs(d - ref)) < 1e-3 * np.max(np.abs(ref)), np.max(np.abs(d - ref))
