"""Which MN-major descriptor stride convention does tcgen05 use (no swizzle)?  Runs the
prb_debug_tc_gemm_major self-test for every (a_mn, b_mn, hyp) and prints the max error vs numpy."""
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2112_05923_b200 import podracer as pr  # noqa: E402

ctx = pr.Context(0)
rng = np.random.default_rng(0)
for K, N in ((64, 64), (128, 144), (32, 16)):
    A = rng.normal(size=(128, K)).astype(np.float32)
    B = rng.normal(size=(N, K)).astype(np.float32)
    bf = lambda x: (x.view(np.uint32) + 0x7FFF + ((x.view(np.uint32) >> 16) & 1) & 0xFFFF0000).view(np.float32)
    ref = bf(A).astype(np.float64) @ bf(B).astype(np.float64).T
    for a_mn in (0, 1):
        for b_mn in (0, 1):
            for hyp in (0, 1):
                D = np.zeros((128, N), np.float32)
                ctx.lib.prb_debug_tc_gemm_major(ctx.h, K, N, a_mn, b_mn, hyp, A.ctypes.data_as(C.POINTER(C.c_float)),
                                                B.ctypes.data_as(C.POINTER(C.c_float)),
                                                D.ctypes.data_as(C.POINTER(C.c_float)))
                err = float(np.max(np.abs(D - ref)))
                print(f"K={K} N={N} a_mn={a_mn} b_mn={b_mn} hyp={hyp}: max err {err:.3e}", flush=True)
