"""GPU: the tcgen05 / TMEM building block (descriptor layout, MMA, TMEM loads)
against a numpy fp32 GEMM of the same bf16-rounded operands."""
import ctypes as C

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def bf16(x):
    b = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32)
    r = ((b + 0x7FFF + ((b >> 16) & 1)) & 0xFFFF0000).astype(np.uint32)  # round-to-nearest-even
    return r.view(np.float32)


@pytest.mark.parametrize("K,N", [(16, 16), (32, 128), (64, 64), (128, 256), (192, 32)])
def test_tc_gemm(K, N):
    from paper_2112_05923_b200 import podracer as pr
    ctx = pr.Context(0)
    rng = np.random.default_rng(K * 7 + N)
    A = rng.normal(size=(128, K)).astype(np.float32)
    B = rng.normal(size=(N, K)).astype(np.float32)
    D = np.zeros((128, N), dtype=np.float32)
    f = C.POINTER(C.c_float)
    ctx.lib.prb_debug_tc_gemm(ctx.h, K, N, A.ctypes.data_as(f), B.ctypes.data_as(f), D.ctypes.data_as(f))
    exp = bf16(A).astype(np.float64) @ bf16(B).astype(np.float64).T
    assert np.allclose(D, exp, rtol=1e-4, atol=1e-4 * np.sqrt(K)), np.max(np.abs(D - exp))
