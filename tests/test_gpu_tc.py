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


def test_trade_math_bit_exact():
    """The fused stock rollout's conversion- and division-free trade arithmetic
    (stock_env.cuh: desired_qty_f32, buy_qty_nodiv) against the reference
    expressions stock_env.hpp:83-97 evaluated in IEEE double, on random inputs and
    on adversarial ones: products and quotients exactly at, and one ulp either
    side of, integers; zero / negative balances; NaN and out-of-range actions."""
    from paper_2112_05923_b200 import podracer as pr
    ctx = pr.Context(0)
    rng = np.random.default_rng(2112)
    mt, cost = 100.0, 1e-3
    n = 1 << 18
    act = rng.uniform(-1.5, 1.5, n).astype(np.float32)
    # actions whose product with max_trade is an integer, and their fp32 neighbours
    k = rng.integers(-100, 101, n // 4)
    exact = (k / mt).astype(np.float32)
    act[: n // 4] = exact
    act[n // 4: n // 2] = np.nextafter(exact, np.float32(np.inf))
    act[n // 2: 3 * n // 4] = np.nextafter(exact, np.float32(-np.inf))
    act[:8] = [np.nan, np.inf, -np.inf, 0.0, -0.0, 1.0, -1.0, 1e-30]
    price = rng.uniform(10.0, 200.0, n)
    pc = price * (1.0 + cost)
    bal = rng.uniform(0.0, 2.0e6, n)
    m = rng.integers(0, 120, n).astype(np.float64)
    q = n // 8  # balances at an exact multiple of pc (rounded), and 1-2 ulp either side
    bal[:q] = m[:q] * pc[:q]
    bal[q:2 * q] = np.nextafter(m[q:2 * q] * pc[q:2 * q], np.inf)
    bal[2 * q:3 * q] = np.nextafter(m[2 * q:3 * q] * pc[2 * q:3 * q], -np.inf)
    bal[3 * q:4 * q] = np.nextafter(np.nextafter(m[3 * q:4 * q] * pc[3 * q:4 * q], -np.inf), -np.inf)
    bal[4 * q:4 * q + 64] = rng.uniform(-1e4, 0.0, 64)
    bal[4 * q + 64:4 * q + 96] = 0.0
    desired = np.zeros(n, np.int32)
    buy = np.zeros(n)
    buy_i = np.zeros(n, np.int32)
    f, d64, i32 = C.POINTER(C.c_float), C.POINTER(C.c_double), C.POINTER(C.c_int32)
    ctx.lib.prb_debug_trade_math(ctx.h, n, act.ctypes.data_as(f), mt, bal.ctypes.data_as(d64),
                                 price.ctypes.data_as(d64), cost, desired.ctypes.data_as(i32),
                                 buy.ctypes.data_as(d64), buy_i.ctypes.data_as(i32))
    with np.errstate(invalid="ignore"):
        want_d = np.trunc(np.clip(act.astype(np.float64), -1.0, 1.0) * mt)
    want_d = np.where(np.isnan(want_d), 0.0, want_d)
    assert np.array_equal(desired, want_d.astype(np.int32))
    afford = np.floor(bal / (price * (1.0 + cost)))
    want_b = np.minimum(want_d, np.maximum(afford, 0.0))
    sel = want_d > 0
    assert sel.sum() > n // 4
    assert np.array_equal(buy[sel], want_b[sel])
    assert np.array_equal(buy_i[sel], want_b[sel].astype(np.int32))
