"""ctypes binding of libprb.so (the prb_* C ABI declared in include/prb.h).

The library is built in-tree by ``__graft_entry__.build()`` (csrc/Makefile,
sm_100a).  There is no fallback: if the shared object is missing or fails to
load, every entry point raises -- the product path never degrades to CPU.
"""
from __future__ import annotations

import ctypes as C
import os
import threading

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("PRB_LIB_PATH") or os.path.join(_HERE, "libprb.so")  # override: A/B builds

_lock = threading.Lock()
_lib = None


class PodracerError(RuntimeError):
    """Base of the reference's exception family (common.hpp:19-71)."""


class DimensionError(PodracerError):
    pass


class NumericError(PodracerError):
    pass


class UsageError(PodracerError):
    pass


class FormatError(PodracerError):
    pass


class DataError(PodracerError):
    pass


class ConfigError(PodracerError):
    pass


class CorruptionError(PodracerError):
    pass


class VersionError(PodracerError):
    pass


class DomainError(PodracerError):
    pass


class DeviceError(PodracerError):
    pass


ERRORS = {1: DimensionError, 2: NumericError, 3: UsageError, 4: FormatError, 5: DataError, 6: ConfigError,
          7: CorruptionError, 8: VersionError, 9: DomainError, 10: DeviceError}

P = C.c_void_p
SZ = C.c_size_t
U64 = C.c_uint64
I64 = C.c_int64
D = C.c_double
I = C.c_int
pD = C.POINTER(C.c_double)
pF = C.POINTER(C.c_float)
pU8 = C.POINTER(C.c_uint8)
pU64 = C.POINTER(C.c_uint64)
pI64 = C.POINTER(C.c_int64)
pI32 = C.POINTER(C.c_int32)
pSZ = C.POINTER(C.c_size_t)


class StockConfig(C.Structure):  # prb_stock_config == StockConfig stock_env.hpp:15-19
    _fields_ = [("initial_capital", D), ("max_trade_shares", D), ("cost_rate", D)]


class EnvSpec(C.Structure):  # prb_env_spec == EnvSpec env.hpp:16-34
    _fields_ = [("state_dim", SZ), ("action_dim", SZ), ("max_episode_steps", SZ), ("reward_target", D),
                ("action_low", pD), ("action_high", pD)]


class PpoConfig(C.Structure):  # prb_ppo_config == PpoConfig ppo.hpp:18-27
    _fields_ = [("gamma", D), ("gae_lambda", D), ("clip_eps", D), ("entropy_coef", D), ("value_coef", D),
                ("epochs_per_update", U64), ("minibatch_size", U64), ("buffer_size", U64), ("learning_rate", D)]


class PpoStats(C.Structure):  # PpoUpdateStats ppo.hpp:198-203
    _fields_ = [("mean_policy_loss", D), ("mean_value_loss", D), ("mean_entropy", D), ("minibatches", U64)]


# name -> (restype, argtypes); int-returning functions are status-checked.
SIGNATURES = {
    "prb_last_error": (C.c_char_p, []),
    "prb_version": (I, []),
    "prb_splitmix64": (U64, [U64]),
    "prb_derive_seed": (U64, [U64, pU64, I]),
    "prb_ctx_create": (I, [I, C.POINTER(P)]),
    "prb_ctx_destroy": (I, [P]),
    "prb_ctx_synchronize": (I, [P]),
    "prb_ctx_stream": (P, [P]),
    "prb_device_alloc": (I, [P, SZ, C.POINTER(P)]),
    "prb_device_free": (I, [P, P]),
    "prb_memcpy_h2d": (I, [P, P, P, SZ]),
    "prb_memcpy_d2h": (I, [P, P, P, SZ]),
    "prb_memcpy_h2d_async": (I, [P, P, P, SZ]),
    "prb_memcpy_d2h_async": (I, [P, P, P, SZ]),
    "prb_market_synthetic": (I, [U64, I, SZ, pD, pD, pD, pD, pD]),
    "prb_compute_indicators": (I, [pD, pD, pD, SZ, I, pD]),
    "prb_market_create": (I, [P, pD, pD, SZ, I, C.POINTER(P)]),
    "prb_market_destroy": (I, [P]),
    "prb_vecenv_create_stock": (I, [P, C.POINTER(StockConfig), SZ, SZ, SZ, C.POINTER(P)]),
    "prb_vecenv_create_pointmass": (I, [P, SZ, C.POINTER(P)]),
    "prb_vecenv_destroy": (I, [P]),
    "prb_vecenv_spec": (I, [P, C.POINTER(EnvSpec)]),
    "prb_vecenv_num_envs": (SZ, [P]),
    "prb_vecenv_states_device": (P, [P]),
    "prb_vecenv_reset": (I, [P, U64, P]),
    "prb_vecenv_step": (I, [P, P, P, P, P, P, P]),
    "prb_vecenv_reset_host": (I, [P, U64, pD]),
    "prb_vecenv_step_host": (I, [P, pD, pD, pD, pU8, pD, pD, pU64]),
    "prb_vecenv_states_host": (I, [P, pD]),
    "prb_vecenv_step_counts_host": (I, [P, pU64]),
    "prb_agent_create": (I, [P, SZ, SZ, pSZ, I, C.POINTER(P)]),
    "prb_agent_destroy": (I, [P]),
    "prb_agent_param_count": (SZ, [P]),
    "prb_agent_set_host": (I, [P, pD, pD, pD, I64, D]),
    "prb_agent_get_host": (I, [P, pD, pD, pD, pI64]),
    "prb_agent_copy": (I, [P, P]),
    "prb_agent_params_device": (P, [P]),
    "prb_artifact_init": (I, [SZ, SZ, U64, pSZ, I, pD, pSZ]),
    "prb_policy_sample": (I, [P, P, SZ, U64, U64, P, P, P, P]),
    "prb_policy_sample_eps": (I, [P, P, SZ, P, P, P, P]),
    "prb_policy_mean": (I, [P, P, SZ, P]),
    "prb_policy_log_prob": (I, [P, P, P, SZ, P]),
    "prb_critic_value": (I, [P, P, SZ, P]),
    "prb_rollout_create": (I, [P, SZ, C.POINTER(P)]),
    "prb_rollout_create_raw": (I, [P, SZ, SZ, SZ, SZ, C.POINTER(P)]),
    "prb_rollout_destroy": (I, [P]),
    "prb_rollout_collect": (I, [P, P, P, U64]),
    "prb_ctx_profile": (I, [P, I]),
    "prb_ctx_profile_read": (I, [P, I, pD, pU64]),
    "prb_rollout_set_mode": (I, [P, I]),
    "prb_rollout_collect_pods": (I, [C.POINTER(P), C.POINTER(P), C.POINTER(P), SZ, pU64]),
    "prb_rollout_device_fields": (I, [P] + [C.POINTER(P)] * 7),
    "prb_rollout_download": (I, [P, pD, pD, pD, pD, pU8, pD, pD]),
    "prb_rollout_upload": (I, [P, pD, pD, pD, pD, pU8, pD, pD]),
    "prb_rollout_download_chunks": (I, [P, pU64, SZ, pD, pD, pD, pD, pU8, pD, pD, pD, pD]),
    "prb_gae_stats": (I, [P, pD, pD]),
    "prb_gae": (I, [P, D, D, I]),
    "prb_gae_download": (I, [P, pD, pD]),
    "prb_rollout_set_advantages": (I, [P, pD, pD]),
    "prb_compute_gae": (I, [P, P, P, P, P, SZ, SZ, D, D, P, P]),
    "prb_ppo_update": (I, [P, P, C.POINTER(PpoConfig), U64, pU64, P, C.POINTER(PpoStats)]),
    "prb_ppo_loss_grads": (I, [P, P, pU64, SZ, C.POINTER(PpoConfig), pD, pD]),
    "prb_ppo_update_learners": (I, [C.POINTER(P), C.POINTER(P), SZ, C.POINTER(PpoConfig), pU64, C.POINTER(P),
                                    C.POINTER(PpoStats)]),
    "prb_adam_step_host": (I, [P, pD]),
    "prb_adam_step_device": (I, [P, P]),
    "prb_evaluate": (I, [P, P, U64, I, pD, pD, pD, pU64]),
    "prb_evaluate_pods": (I, [C.POINTER(P), C.POINTER(P), SZ, pU64, I, pD, pD, pD, pU64]),
    "prb_fuse_parameters": (I, [C.POINTER(P), SZ, P]),
    "prb_leaderboard_rank": (I, [P, P, P, SZ, SZ, P, P]),
    "prb_leaderboard_rank_host": (I, [P, pD, pU64, SZ, SZ, pI32, pI32]),
    "prb_agent_mutate": (I, [P, U64, D]),
    "prb_agent_set_ppo_mode": (I, [P, I]),
    "prb_agent_init_device": (I, [P, U64, D]),
    "prb_debug_agent_grads": (I, [P, pD]),
    "prb_leaderboard_stats": (I, [C.POINTER(P), SZ, P, P]),
    "prb_leaderboard_stats_host": (I, [C.POINTER(P), SZ, pD, pD]),
    "prb_debug_set_option": (I, [I, I]),
    "prb_checkpoint_encode": (I, [P, I64, U64, C.c_char_p, pD, pU8, SZ, C.POINTER(SZ)]),
    "prb_checkpoint_decode": (I, [P, pU8, SZ, C.POINTER(I64), pU64, C.c_char_p, SZ, pD, C.POINTER(I)]),
    "prb_checkpoint_save": (I, [P, C.c_char_p, I64, U64, C.c_char_p, pD]),
    "prb_checkpoint_load": (I, [P, C.c_char_p, C.POINTER(I64), pU64, C.c_char_p, SZ, pD, C.POINTER(I)]),
    "prb_checkpoint_encode_host": (I, [SZ, SZ, pSZ, I, pD, pD, pD, I64, pD, I64, U64, C.c_char_p, pD, pU8, SZ,
                                       C.POINTER(SZ)]),
    "prb_checkpoint_decode_host": (I, [pU8, SZ, SZ, SZ, pSZ, I, pD, pD, pD, C.POINTER(I64), pD, C.POINTER(I64), pU64,
                                       C.c_char_p, SZ, pD, C.POINTER(I)]),
    "prb_comm_unique_id": (I, [C.POINTER(C.c_uint8)]),
    "prb_comm_init": (I, [P, C.POINTER(C.c_uint8), I, I, C.POINTER(P)]),
    "prb_comm_destroy": (I, [P]),
    "prb_leaderboard_allgather_rank": (I, [P, P, P, P, SZ, SZ, P, P, P, P, P]),
    "prb_agent_broadcast": (I, [P, P, I]),
    "prb_debug_tc_gemm": (I, [P, I, I, pF, pF, pF]),
    "prb_debug_tc_gemm_major": (I, [P, I, I, I, I, I, pF, pF, pF]),
    "prb_debug_trade_math": (I, [P, SZ, pF, D, pD, pD, D, pI32, pD, pI32]),
}

UNCHECKED = {"prb_last_error", "prb_version", "prb_splitmix64", "prb_derive_seed", "prb_ctx_stream",
             "prb_vecenv_num_envs", "prb_vecenv_states_device", "prb_agent_param_count", "prb_agent_params_device"}


class _Checked:
    def __init__(self, lib, name, fn):
        self._lib, self._name, self._fn = lib, name, fn

    def __call__(self, *args):
        rc = self._fn(*args)
        if rc != 0:
            msg = self._lib.prb_last_error().decode(errors="replace")
            raise ERRORS.get(rc, PodracerError)(f"{self._name}: {msg}")
        return rc


class Lib:
    def __init__(self, cdll):
        self._cdll = cdll
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(cdll, name)
            fn.restype = res
            fn.argtypes = args
            setattr(self, name, fn if (name in UNCHECKED or res is not I) else _Checked(cdll, name, fn))
        self.prb_last_error = cdll.prb_last_error

    @property
    def path(self):
        return self._cdll._name


def lib() -> Lib:
    """Load libprb.so (raises if it was not built -- no fallback)."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise ImportError(f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'`")
            _lib = Lib(C.CDLL(LIB_PATH))
        return _lib
