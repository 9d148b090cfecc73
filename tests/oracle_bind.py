"""ctypes bindings for the CHECKER libraries (test infrastructure only).

* ``orc``  -- oracle/liboracle.so, the plain-C restatement (podracer_oracle.c).
* ``ref``  -- oracle/_ref/libpodracer_ref_exact.so, the unmodified reference
  headers behind a C shim (built only where /root/reference exists; the .so
  travels to the GPU box with the snapshot).  ``ref`` is None when absent.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg use these.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ORACLE_SO = os.path.join(ROOT, "oracle", "liboracle.so")
REF_EXACT_SO = os.path.join(ROOT, "oracle", "_ref", "libpodracer_ref_exact.so")
REF_BENCH_SO = os.path.join(ROOT, "oracle", "_ref", "libpodracer_ref_bench.so")

D = C.POINTER(C.c_double)
U64 = C.POINTER(C.c_uint64)
I64 = C.POINTER(C.c_int64)
SZ = C.POINTER(C.c_size_t)
U8 = C.POINTER(C.c_uint8)
I32 = C.POINTER(C.c_int)


def ptr(a: np.ndarray | None, t=D):
    if a is None:
        return None
    assert a.flags["C_CONTIGUOUS"], "arrays passed to the checker must be C-contiguous"
    return a.ctypes.data_as(t)


class MT64(C.Structure):
    _fields_ = [("mt", C.c_uint64 * 312), ("idx", C.c_int)]


class StockCfg(C.Structure):
    _fields_ = [("initial_capital", C.c_double), ("max_trade_shares", C.c_double), ("cost_rate", C.c_double)]


class PpoCfg(C.Structure):
    _fields_ = [("gamma", C.c_double), ("gae_lambda", C.c_double), ("clip_eps", C.c_double),
                ("entropy_coef", C.c_double), ("value_coef", C.c_double), ("epochs_per_update", C.c_uint64),
                ("minibatch_size", C.c_uint64), ("buffer_size", C.c_uint64), ("learning_rate", C.c_double)]


def _load(path):
    if not os.path.exists(path):
        return None
    return C.CDLL(path)


def load_oracle():
    lib = _load(ORACLE_SO)
    if lib is None:
        raise RuntimeError(f"checker library missing: {ORACLE_SO} (run `make -C oracle`)")
    lib.orc_splitmix64.restype = C.c_uint64
    lib.orc_splitmix64.argtypes = [C.c_uint64]
    lib.orc_derive_seed.restype = C.c_uint64
    lib.orc_derive_seed.argtypes = [C.c_uint64, U64, C.c_int]
    lib.orc_mt64_seed.argtypes = [C.POINTER(MT64), C.c_uint64]
    lib.orc_mt64_next.restype = C.c_uint64
    lib.orc_mt64_next.argtypes = [C.POINTER(MT64)]
    lib.orc_uniform_real.restype = C.c_double
    lib.orc_uniform_real.argtypes = [C.POINTER(MT64), C.c_double, C.c_double]
    lib.orc_philox4x32_10.argtypes = [C.c_uint32, C.c_uint32, C.POINTER(C.c_uint32), C.POINTER(C.c_uint32)]
    lib.orc_stock_env_step.restype = C.c_int
    lib.orc_stock_env_step.argtypes = [D, D, SZ, D, D, C.c_size_t, C.c_int, C.POINTER(StockCfg), D, I32]
    lib.orc_stock_observation.argtypes = [C.c_double, D, C.c_size_t, D, D, C.c_size_t, C.c_int,
                                          C.POINTER(StockCfg), C.c_size_t, D]
    lib.orc_stock_vec_reset.argtypes = [C.c_size_t, C.c_int, C.POINTER(StockCfg), C.c_size_t, D, D, SZ, SZ, D]
    lib.orc_stock_vec_step.restype = C.c_int
    lib.orc_stock_vec_step.argtypes = [C.c_size_t, C.c_int, C.POINTER(StockCfg), C.c_size_t, C.c_size_t, D, D,
                                       C.c_size_t, D, D, SZ, SZ, D, D, D, D, U8, D, D, U64]
    lib.orc_pointmass_step.argtypes = [D, D, C.c_uint64, D, D, I32]
    lib.orc_pointmass_reset.argtypes = [C.POINTER(MT64), D]
    lib.orc_pm_vec_reset.argtypes = [C.c_size_t, C.c_uint64, C.POINTER(MT64), D, U64, D]
    lib.orc_pm_vec_reset_subset.argtypes = [C.c_size_t, U64, C.c_uint64, C.POINTER(MT64), D, U64, D]
    lib.orc_pm_vec_step.argtypes = [C.c_size_t, C.POINTER(MT64), D, U64, D, D, D, U8, D, D, U64]
    lib.orc_mlp_param_count.restype = C.c_size_t
    lib.orc_mlp_param_count.argtypes = [SZ, C.c_int]
    lib.orc_mlp_forward.argtypes = [D, SZ, C.c_int, D, C.c_size_t, D, D]
    lib.orc_gaussian_row_log_prob.restype = C.c_double
    lib.orc_gaussian_row_log_prob.argtypes = [D, C.c_int, D, D]
    lib.orc_policy_sample_eps.argtypes = [D, SZ, C.c_int, D, D, C.c_size_t, D, D, D]
    lib.orc_policy_entropy.restype = C.c_double
    lib.orc_policy_entropy.argtypes = [D, C.c_int]
    lib.orc_compute_gae.argtypes = [D, D, U8, C.c_size_t, C.c_double, C.c_double, C.c_double, D, D]
    lib.orc_buffer_advantages.restype = C.c_int
    lib.orc_buffer_advantages.argtypes = [D, D, U8, C.c_size_t, SZ, SZ, D, C.c_size_t, C.c_double, C.c_double,
                                          C.c_int, D, D]
    lib.orc_ppo_loss_grads.restype = C.c_int
    lib.orc_ppo_loss_grads.argtypes = [D, SZ, C.c_int, SZ, C.c_int, D, D, D, D, D, C.c_size_t,
                                       C.POINTER(PpoCfg), D, D]
    lib.orc_adam_step.restype = C.c_int
    lib.orc_adam_step.argtypes = [D, D, D, D, I64, C.c_size_t, C.c_double, C.c_double, C.c_double, C.c_double]
    lib.orc_ppo_update.restype = C.c_int
    lib.orc_ppo_update.argtypes = [D, D, D, I64, SZ, C.c_int, SZ, C.c_int, D, D, D, D, U8, D, C.c_size_t, C.c_int,
                                   SZ, SZ, D, C.c_size_t, C.POINTER(PpoCfg), U64, D]
    lib.orc_fuse.argtypes = [C.POINTER(D), C.POINTER(D), C.POINTER(D), I64, C.c_size_t, C.c_size_t, D, D, D, I64]
    lib.orc_population_stats.restype = None
    lib.orc_population_stats.argtypes = [C.POINTER(D), C.c_size_t, C.c_size_t, D, D]
    lib.orc_leaderboard_update.restype = C.c_int
    lib.orc_leaderboard_update.argtypes = [D, U64, I64, SZ, C.c_size_t, U64, C.c_double, C.c_int64]
    lib.orc_compute_indicators.restype = C.c_int
    lib.orc_compute_indicators.argtypes = [D, D, D, C.c_size_t, C.c_int, D]
    return lib


def load_ref(path: str = REF_EXACT_SO):
    lib = _load(path)
    if lib is None:
        return None
    lib.ref_derive_seed.restype = C.c_uint64
    lib.ref_derive_seed.argtypes = [C.c_uint64, U64, C.c_int]
    lib.ref_uniform_real_draws.argtypes = [C.c_uint64, C.c_double, C.c_double, C.c_size_t, D]
    lib.ref_mt64_draws.argtypes = [C.c_uint64, C.c_size_t, U64]
    lib.ref_stock_env_step.restype = C.c_int
    lib.ref_stock_env_step.argtypes = [D, D, SZ, D, D, C.c_size_t, C.c_int, D, D, I32]
    lib.ref_stock_vec_create.restype = C.c_void_p
    lib.ref_stock_vec_create.argtypes = [D, D, C.c_size_t, C.c_int, D, C.c_size_t, C.c_size_t, C.c_size_t]
    lib.ref_pm_vec_create.restype = C.c_void_p
    lib.ref_pm_vec_create.argtypes = [C.c_size_t]
    lib.ref_vec_destroy.argtypes = [C.c_void_p]
    lib.ref_vec_reset.restype = C.c_int
    lib.ref_vec_reset.argtypes = [C.c_void_p, C.c_uint64, D]
    lib.ref_vec_step.restype = C.c_int
    lib.ref_vec_step.argtypes = [C.c_void_p, D, C.c_size_t, D, D, U8, D, D, U64]
    lib.ref_vec_step_counts.argtypes = [C.c_void_p, U64]
    lib.ref_pointmass_step.restype = C.c_int
    lib.ref_pointmass_step.argtypes = [D, D, C.c_uint64, D, D, I32]
    lib.ref_compute_indicators.restype = C.c_int
    lib.ref_compute_indicators.argtypes = [D, D, D, C.c_size_t, C.c_int, D]
    lib.ref_mlp_forward.restype = C.c_int
    lib.ref_mlp_forward.argtypes = [D, SZ, C.c_int, D, C.c_size_t, D]
    lib.ref_gaussian_row_log_prob.restype = C.c_double
    lib.ref_gaussian_row_log_prob.argtypes = [D, C.c_int, D, D]
    lib.ref_adam_step.restype = C.c_int
    lib.ref_adam_step.argtypes = [D, D, D, D, I64, C.c_size_t, C.c_double]
    lib.ref_artifact_init.restype = C.c_size_t
    lib.ref_artifact_init.argtypes = [C.c_size_t, C.c_size_t, C.c_uint64, C.c_double, SZ, C.c_int, D]
    lib.ref_compute_gae.restype = C.c_int
    lib.ref_compute_gae.argtypes = [D, D, U8, C.c_size_t, C.c_double, C.c_double, C.c_double, D, D]
    lib.ref_buffer_advantages.restype = C.c_int
    lib.ref_buffer_advantages.argtypes = [D, D, U8, C.c_size_t, SZ, SZ, D, C.c_size_t, C.c_double, C.c_double,
                                          C.c_int, D, D]
    lib.ref_ppo_loss_grads.restype = C.c_int
    lib.ref_ppo_loss_grads.argtypes = [D, C.c_size_t, C.c_size_t, SZ, C.c_int, D, D, D, D, D, C.c_size_t, D, D, D]
    lib.ref_ppo_permutations.argtypes = [C.c_uint64, C.c_size_t, C.c_size_t, U64]
    lib.ref_ppo_update.restype = C.c_int
    lib.ref_ppo_update.argtypes = [D, D, D, I64, C.c_size_t, C.c_size_t, SZ, C.c_int, D, D, D, D, U8, D,
                                   C.c_size_t, SZ, SZ, D, C.c_size_t, D, C.c_uint64, D]
    lib.ref_fuse.restype = C.c_int
    lib.ref_fuse.argtypes = [C.POINTER(D), C.POINTER(D), C.POINTER(D), I64, C.c_size_t, C.c_size_t, C.c_size_t,
                             SZ, C.c_int, D, D, D, I64]
    lib.ref_leaderboard_stats.restype = C.c_int
    lib.ref_leaderboard_stats.argtypes = [D, D, I64, C.c_size_t, C.c_size_t, C.c_size_t, C.c_size_t, SZ, C.c_int,
                                          I64, SZ, D, D]
    lib.ref_leaderboard_sequence.restype = C.c_int
    lib.ref_leaderboard_sequence.argtypes = [D, I64, C.c_size_t, C.c_size_t, I64, D, SZ, I64]
    lib.ref_checkpoint_encode.restype = C.c_size_t
    lib.ref_checkpoint_encode.argtypes = [D, D, D, C.c_int64, D, C.c_size_t, C.c_size_t, SZ, C.c_int, C.c_int64,
                                          C.c_uint64, C.c_char_p, D, U8]
    lib.ref_checkpoint_decode.restype = C.c_int
    lib.ref_checkpoint_decode.argtypes = [U8, C.c_size_t, D, D, D, I64, I64, U64]
    lib.ref_synthetic_market.restype = None
    lib.ref_synthetic_market.argtypes = [C.c_uint64, C.c_int, C.c_size_t, D, D, D]
    lib.ref_bench_ppo.restype = C.c_double
    lib.ref_bench_ppo.argtypes = [D, C.c_size_t, C.c_size_t, SZ, C.c_int, C.c_size_t, C.c_size_t, C.c_size_t,
                                  C.c_size_t, C.c_uint64]
    lib.ref_bench_collect.restype = C.c_double
    lib.ref_bench_collect.argtypes = [D, D, C.c_size_t, C.c_int, C.c_size_t, C.c_size_t, C.c_size_t, C.c_size_t,
                                      C.c_size_t, D, SZ, C.c_int, C.c_uint64]
    lib.ref_bench_env_step.restype = C.c_double
    lib.ref_bench_env_step.argtypes = [D, D, C.c_size_t, C.c_int, C.c_size_t, C.c_size_t, C.c_size_t, C.c_size_t,
                                       C.c_size_t]
    return lib


# ---------------------------------------------------------------------------
# Convenience wrappers used by several tests.
# ---------------------------------------------------------------------------

def derive_seed(lib, base: int, *tags: int) -> int:
    arr = (C.c_uint64 * max(1, len(tags)))(*tags)
    fn = lib.orc_derive_seed if hasattr(lib, "orc_derive_seed") else lib.ref_derive_seed
    return int(fn(C.c_uint64(base), arr, len(tags)))


def synthetic_market_np(K: int, T: int, seed: int = 2112):
    """Numpy-free description is in BASELINE.md §3; the generator itself is the
    product's (prb_market_synthetic).  This helper is a small independent
    random-walk market for checker-only tests (not used on the product path)."""
    rng = np.random.default_rng(seed)
    p0 = rng.uniform(10.0, 200.0, size=K)
    steps = np.exp(1e-3 * rng.standard_normal(size=(K, T - 1)))
    close = np.empty((K, T))
    close[:, 0] = p0
    close[:, 1:] = p0[:, None] * np.cumprod(steps, axis=1)
    high = close * 1.001
    low = close * 0.999
    return np.ascontiguousarray(close), np.ascontiguousarray(high), np.ascontiguousarray(low)


def indicators(lib, high, low, close):
    K, T = close.shape
    out = np.zeros((4, K, T))
    fn = lib.orc_compute_indicators if hasattr(lib, "orc_compute_indicators") else lib.ref_compute_indicators
    rc = fn(ptr(high), ptr(low), ptr(close), T, K, ptr(out))
    assert rc == 0
    return out


def population_stats(orc, entries):
    """orc_population_stats over a list of flat f64 param vectors in board order."""
    n = len(entries)
    P = len(entries[0]) if n else 0
    arrs = [np.ascontiguousarray(e, dtype=np.float64) for e in entries]
    ptrs = (D * max(n, 1))(*[ptr(a) for a in arrs])
    mean, var = np.zeros(P), np.zeros(P)
    orc.orc_population_stats(ptrs, n, P, ptr(mean), ptr(var))
    return mean, var
