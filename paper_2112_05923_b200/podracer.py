"""Python host mirror of the reference's hot-path API over the prb_* C ABI.

Names, argument meaning and error behaviour follow the reference C++ API
(SURVEY.md §8b): ``VectorizedEnvironment.reset/step`` (env.hpp:167-249),
``policy_sample`` (nn.hpp:250), ``TransitionBuffer``/``worker_collect``
(buffer.hpp, pod.hpp:95), ``buffer_advantages`` (ppo.hpp:212), ``ppo_update``
(ppo.hpp:249), ``fuse_parameters`` (pod.hpp:141), ``leaderboard_update``
(tournament.hpp:104).  Every call goes through libprb.so; there is no CPU
implementation here.  Host arrays are numpy float64 in the reference's
Tensor2 layouts; device-resident variants take/return ``DeviceArray``.
"""
from __future__ import annotations

import ctypes as C
import sys
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np

from . import _lib
from ._lib import (ConfigError, DataError, DimensionError, NumericError, PodracerError, UsageError, EnvSpec,
                   PpoConfig as _PpoConfigC, PpoStats as _PpoStatsC, StockConfig as _StockConfigC)

__all__ = ["Context", "DeviceArray", "MarketData", "StockConfig", "VectorizedEnvironment", "VecStepResult",
           "VecStepInfo", "Agent", "artifact_init", "Rollout", "PpoConfig", "PpoUpdateStats", "ppo_update",
           "fuse_parameters", "leaderboard_rank", "derive_seed", "synthetic_market", "compute_indicators",
           "DimensionError", "NumericError", "UsageError", "ConfigError", "DataError", "PodracerError"]


def _p(a: np.ndarray, ct):
    return a.ctypes.data_as(C.POINTER(ct))


def derive_seed(base: int, *tags: int) -> int:
    """common.hpp:88-93."""
    arr = (C.c_uint64 * max(1, len(tags)))(*tags)
    return int(_lib.lib().prb_derive_seed(base, arr, len(tags)))


class Context:
    """One device + one CUDA stream (the unit a reference worker thread owns)."""

    def __init__(self, device: int = 0):
        self.lib = _lib.lib()
        h = C.c_void_p()
        self.lib.prb_ctx_create(device, C.byref(h))
        self.h = h
        self.device = device

    def synchronize(self):
        self.lib.prb_ctx_synchronize(self.h)

    @property
    def stream(self) -> int:
        return int(self.lib.prb_ctx_stream(self.h) or 0)

    def alloc(self, shape, dtype=np.float32) -> "DeviceArray":
        return DeviceArray(self, shape, dtype)

    def close(self):
        if self.h:
            self.lib.prb_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        if sys.is_finalizing():  # interpreter teardown: arbitrary order (a context may already be gone)
            return
        try:
            self.close()
        except Exception:
            pass


class DeviceArray:
    """A cudaMalloc'd buffer owned by the library's allocator."""

    def __init__(self, ctx: Context, shape, dtype=np.float32):
        self.ctx = ctx
        self.shape = tuple(int(s) for s in (shape if isinstance(shape, (tuple, list)) else (shape,)))
        self.dtype = np.dtype(dtype)
        self.nbytes = int(np.prod(self.shape, dtype=np.int64)) * self.dtype.itemsize
        p = C.c_void_p()
        ctx.lib.prb_device_alloc(ctx.h, max(self.nbytes, 1), C.byref(p))
        self.ptr = p.value

    @classmethod
    def from_numpy(cls, ctx: Context, a: np.ndarray, dtype=None) -> "DeviceArray":
        a = np.ascontiguousarray(a, dtype=dtype or a.dtype)
        d = cls(ctx, a.shape, a.dtype)
        d.upload(a)
        return d

    def upload(self, a: np.ndarray):
        a = np.ascontiguousarray(a, dtype=self.dtype)
        assert a.nbytes == self.nbytes, (a.shape, self.shape)
        self.ctx.lib.prb_memcpy_h2d(self.ctx.h, self.ptr, a.ctypes.data, self.nbytes)

    def numpy(self) -> np.ndarray:
        out = np.empty(self.shape, dtype=self.dtype)
        self.ctx.lib.prb_memcpy_d2h(self.ctx.h, out.ctypes.data, self.ptr, self.nbytes)
        return out

    def free(self):
        if self.ptr:
            self.ctx.lib.prb_device_free(self.ctx.h, self.ptr)
            self.ptr = None

    def __del__(self):
        if sys.is_finalizing():  # interpreter teardown: arbitrary order (a context may already be gone)
            return
        try:
            self.free()
        except Exception:
            pass


# ---------------------------------------------------------------------------
# Market data (market.hpp) -- the format the env kernel consumes.
# ---------------------------------------------------------------------------

def synthetic_market(K: int = 30, T: int = 2048, seed: int = 2112):
    """BASELINE.md §3 synthetic OHLCV; returns dict of [K][T] float64 arrays."""
    lib = _lib.lib()
    out = {k: np.zeros((K, T)) for k in ("open", "high", "low", "close", "volume")}
    lib.prb_market_synthetic(seed, K, T, *[_p(out[k], C.c_double) for k in ("open", "high", "low", "close", "volume")])
    return out


def compute_indicators(high: np.ndarray, low: np.ndarray, close: np.ndarray) -> np.ndarray:
    """compute_indicators market.hpp:373-392 -> [4][K][T] (macd, rsi_14, cci_30, sma_20)."""
    K, T = close.shape
    h, l, c = (np.ascontiguousarray(x, dtype=np.float64) for x in (high, low, close))
    out = np.zeros((4, K, T))
    _lib.lib().prb_compute_indicators(_p(h, C.c_double), _p(l, C.c_double), _p(c, C.c_double), T, K,
                                      _p(out, C.c_double))
    return out


class MarketData:
    """Device-resident MarketData (prices f64 + indicators) for StockTradingEnv."""

    def __init__(self, ctx: Context, close: np.ndarray, indicators: Optional[np.ndarray]):
        self.ctx = ctx
        self.close = np.ascontiguousarray(close, dtype=np.float64)
        self.K, self.T = self.close.shape
        self.indicators = None if indicators is None else np.ascontiguousarray(indicators, dtype=np.float64)
        h = C.c_void_p()
        ctx.lib.prb_market_create(ctx.h, _p(self.close, C.c_double),
                                  None if self.indicators is None else _p(self.indicators, C.c_double),
                                  self.T, self.K, C.byref(h))
        self.h = h

    @classmethod
    def synthetic(cls, ctx: Context, K: int = 30, T: int = 2048, seed: int = 2112) -> "MarketData":
        m = synthetic_market(K, T, seed)
        return cls(ctx, m["close"], compute_indicators(m["high"], m["low"], m["close"]))

    def __del__(self):
        if sys.is_finalizing():  # interpreter teardown: arbitrary order (a context may already be gone)
            return
        try:
            if self.h:
                self.ctx.lib.prb_market_destroy(self.h)
        except Exception:
            pass


@dataclass
class StockConfig:  # stock_env.hpp:15-19
    initial_capital: float = 1_000_000.0
    max_trade_shares: float = 100.0
    cost_rate: float = 0.002


@dataclass
class VecStepInfo:  # env.hpp:153-158
    episode_end: bool = False
    terminal_state: Optional[np.ndarray] = None
    episode_return: float = 0.0
    episode_length: int = 0


@dataclass
class VecStepResult:  # env.hpp:160-165
    next_states: np.ndarray
    rewards: np.ndarray
    dones: np.ndarray
    infos: List[VecStepInfo] = field(default_factory=list)


class VectorizedEnvironment:
    """VectorizedEnvironment (env.hpp:167-249) over device sub-environments."""

    def __init__(self, ctx: Context, handle: C.c_void_p, keepalive=None):
        self.ctx = ctx
        self.h = handle
        self._keep = keepalive
        spec = EnvSpec()
        ctx.lib.prb_vecenv_spec(self.h, C.byref(spec))
        self.state_dim = spec.state_dim
        self.action_dim = spec.action_dim
        self.max_episode_steps = spec.max_episode_steps
        self.reward_target = spec.reward_target
        self.action_low = np.array([spec.action_low[i] for i in range(spec.action_dim)])
        self.action_high = np.array([spec.action_high[i] for i in range(spec.action_dim)])
        self._num_envs = int(ctx.lib.prb_vecenv_num_envs(self.h))

    @classmethod
    def stock(cls, ctx: Context, market: MarketData, cfg: StockConfig, start: int, end: int, num_envs: int):
        h = C.c_void_p()
        c = _StockConfigC(cfg.initial_capital, cfg.max_trade_shares, cfg.cost_rate)
        ctx.lib.prb_vecenv_create_stock(market.h, C.byref(c), start, end, num_envs, C.byref(h))
        return cls(ctx, h, keepalive=market)

    @classmethod
    def pointmass(cls, ctx: Context, num_envs: int):
        h = C.c_void_p()
        ctx.lib.prb_vecenv_create_pointmass(ctx.h, num_envs, C.byref(h))
        return cls(ctx, h)

    def num_envs(self) -> int:
        return self._num_envs

    def spec(self):
        return self

    # -- host-buffer API (reference Tensor2 layouts) --
    def reset(self, seed: int) -> np.ndarray:
        out = np.zeros((self._num_envs, self.state_dim))
        self.ctx.lib.prb_vecenv_reset_host(self.h, seed, _p(out, C.c_double))
        return out

    def states(self) -> np.ndarray:
        out = np.zeros((self._num_envs, self.state_dim))
        self.ctx.lib.prb_vecenv_states_host(self.h, _p(out, C.c_double))
        return out

    def step_counts(self) -> np.ndarray:
        out = np.zeros(self._num_envs, dtype=np.uint64)
        self.ctx.lib.prb_vecenv_step_counts_host(self.h, _p(out, C.c_uint64))
        return out

    def step(self, actions: np.ndarray) -> VecStepResult:
        actions = np.asarray(actions, dtype=np.float64)
        if actions.ndim != 2 or actions.shape != (self._num_envs, self.action_dim):  # env.hpp:201-205
            raise DimensionError(f"vec_step: actions {list(actions.shape)} vs expected "
                                 f"[{self._num_envs}x{self.action_dim}]")
        actions = np.ascontiguousarray(actions)
        N, S = self._num_envs, self.state_dim
        nxt = np.zeros((N, S)); rew = np.zeros(N); done = np.zeros(N, dtype=np.uint8)
        term = np.zeros((N, S)); tret = np.zeros(N); tlen = np.zeros(N, dtype=np.uint64)
        self.ctx.lib.prb_vecenv_step_host(self.h, _p(actions, C.c_double), _p(nxt, C.c_double), _p(rew, C.c_double),
                                          _p(done, C.c_uint8), _p(term, C.c_double), _p(tret, C.c_double),
                                          _p(tlen, C.c_uint64))
        infos = [VecStepInfo(True, term[i].copy(), float(tret[i]), int(tlen[i])) if done[i] else VecStepInfo()
                 for i in range(N)]
        return VecStepResult(nxt, rew, done, infos)

    # -- device-buffer API --
    def reset_device(self, seed: int):
        self.ctx.lib.prb_vecenv_reset(self.h, seed, None)

    def states_device_ptr(self) -> int:
        return int(self.ctx.lib.prb_vecenv_states_device(self.h))

    def step_device(self, d_actions: int, d_reward=None, d_done=None, d_term_obs=None, d_term_ret=None,
                    d_term_len=None):
        self.ctx.lib.prb_vecenv_step(self.h, d_actions, d_reward, d_done, d_term_obs, d_term_ret, d_term_len)

    def __del__(self):
        if sys.is_finalizing():  # interpreter teardown: arbitrary order (a context may already be gone)
            return
        try:
            if self.h:
                self.ctx.lib.prb_vecenv_destroy(self.h)
        except Exception:
            pass


def artifact_init(state_dim: int, action_dim: int, seed: int, hidden: Sequence[int] = (64, 64)) -> np.ndarray:
    """artifact_init artifact.hpp:91-105 -> canonical flat parameter vector (float64)."""
    lib = _lib.lib()
    hid = np.array(hidden, dtype=np.uint64)
    n = C.c_size_t()
    lib.prb_artifact_init(state_dim, action_dim, seed, _p(hid, C.c_size_t), len(hidden), None, C.byref(n))
    flat = np.zeros(n.value)
    lib.prb_artifact_init(state_dim, action_dim, seed, _p(hid, C.c_size_t), len(hidden), _p(flat, C.c_double), None)
    return flat


class Agent:
    """Device AgentArtifact: actor + log_std + critic in the canonical flat
    layout (artifact.hpp:35-51) with Adam state (nn.hpp:144-152)."""

    def __init__(self, ctx: Context, state_dim: int, action_dim: int, hidden: Sequence[int] = (64, 64)):
        self.ctx = ctx
        self.state_dim, self.action_dim, self.hidden = state_dim, action_dim, tuple(hidden)
        hid = np.array(hidden, dtype=np.uint64)
        h = C.c_void_p()
        ctx.lib.prb_agent_create(ctx.h, state_dim, action_dim, _p(hid, C.c_size_t), len(hidden), C.byref(h))
        self.h = h
        self.param_count = int(ctx.lib.prb_agent_param_count(self.h))

    @classmethod
    def init(cls, ctx: Context, state_dim: int, action_dim: int, seed: int, lr: float = 1e-3,
             hidden: Sequence[int] = (64, 64)) -> "Agent":
        a = cls(ctx, state_dim, action_dim, hidden)
        a.set(artifact_init(state_dim, action_dim, seed, hidden), lr=lr)
        return a

    def set(self, flat, m=None, v=None, t: int = 0, lr: float = 1e-3):
        flat = np.ascontiguousarray(flat, dtype=np.float64)
        if flat.size != self.param_count:
            raise DimensionError(f"unflatten_params: {flat.size} values vs {self.param_count} params")
        mm = None if m is None else np.ascontiguousarray(m, dtype=np.float64)
        vv = None if v is None else np.ascontiguousarray(v, dtype=np.float64)
        self.ctx.lib.prb_agent_set_host(self.h, _p(flat, C.c_double), None if mm is None else _p(mm, C.c_double),
                                        None if vv is None else _p(vv, C.c_double), int(t), float(lr))

    def get(self):
        P = self.param_count
        flat, m, v = np.zeros(P), np.zeros(P), np.zeros(P)
        t = C.c_int64()
        self.ctx.lib.prb_agent_get_host(self.h, _p(flat, C.c_double), _p(m, C.c_double), _p(v, C.c_double),
                                        C.byref(t))
        return flat, m, v, t.value

    def flatten_params(self) -> np.ndarray:
        return self.get()[0]

    def init_device(self, seed: int, lr: float = 1e-3) -> "Agent":
        """artifact_init (artifact.hpp:91-105) drawn on the device, bit-exact with the reference."""
        self.ctx.lib.prb_agent_init_device(self.h, seed, lr)
        return self

    def copy_from(self, other: "Agent") -> "Agent":
        """Deep copy of other's params / Adam state into this agent (on the device)."""
        self.ctx.lib.prb_agent_copy(self.h, other.h)
        return self

    def clone(self) -> "Agent":
        b = Agent(self.ctx, self.state_dim, self.action_dim, self.hidden)
        self.ctx.lib.prb_agent_copy(b.h, self.h)
        return b

    def adam_step(self, grads: np.ndarray):
        g = np.ascontiguousarray(grads, dtype=np.float64)
        if g.size != self.param_count:
            raise DimensionError(f"adam_step: params {self.param_count}, grads {g.size}")
        self.ctx.lib.prb_adam_step_host(self.h, _p(g, C.c_double))

    def adam_step_device(self, d_grads: int):
        """adam_step (nn.hpp:164-182) with device fp32 gradients at address d_grads."""
        self.ctx.lib.prb_adam_step_device(self.h, C.c_void_p(d_grads))

    def set_ppo_mode(self, mode: int):
        """0 (default): fp32 SIMT update over the whole GPU; 1: the tensor-core update (8 co-resident CTAs per learner) where the
        shapes allow (what ppo_update_learners always runs)."""
        self.ctx.lib.prb_agent_set_ppo_mode(self.h, int(mode))

    def mutate(self, mutation_seed: int, sigma: float):
        self.ctx.lib.prb_agent_mutate(self.h, mutation_seed, sigma)

    # -- policy (nn.hpp:229-277) on host arrays --
    def _states(self, states):
        s = np.ascontiguousarray(states, dtype=np.float32)
        if s.ndim != 2 or s.shape[1] != self.state_dim:
            raise DimensionError(f"mlp_forward: input {list(s.shape)} vs weights [{self.state_dim}x..]")
        return s

    def policy_sample(self, states, seed: int, counter: int = 0, with_values: bool = False, eps=None):
        s = self._states(states)
        n = s.shape[0]
        ds = DeviceArray.from_numpy(self.ctx, s)
        act = DeviceArray(self.ctx, (n, self.action_dim)); lp = DeviceArray(self.ctx, (n,))
        val = DeviceArray(self.ctx, (n,)) if with_values else None
        if eps is None:
            de = DeviceArray(self.ctx, (n, self.action_dim))
            self.ctx.lib.prb_policy_sample(self.h, ds.ptr, n, seed, counter, act.ptr, lp.ptr,
                                           val.ptr if val else None, de.ptr)
        else:
            de = DeviceArray.from_numpy(self.ctx, np.asarray(eps, dtype=np.float32))
            self.ctx.lib.prb_policy_sample_eps(self.h, ds.ptr, n, de.ptr, act.ptr, lp.ptr, val.ptr if val else None)
        out = dict(actions=act.numpy(), log_probs=lp.numpy(), eps=de.numpy())
        if val:
            out["values"] = val.numpy()
        return out

    def policy_mean(self, states):
        s = self._states(states)
        ds = DeviceArray.from_numpy(self.ctx, s)
        out = DeviceArray(self.ctx, (s.shape[0], self.action_dim))
        self.ctx.lib.prb_policy_mean(self.h, ds.ptr, s.shape[0], out.ptr)
        return out.numpy()

    def log_prob(self, states, actions):
        s = self._states(states)
        ds = DeviceArray.from_numpy(self.ctx, s)
        da = DeviceArray.from_numpy(self.ctx, np.asarray(actions, dtype=np.float32))
        out = DeviceArray(self.ctx, (s.shape[0],))
        self.ctx.lib.prb_policy_log_prob(self.h, ds.ptr, da.ptr, s.shape[0], out.ptr)
        return out.numpy()

    def value(self, states):
        s = self._states(states)
        ds = DeviceArray.from_numpy(self.ctx, s)
        out = DeviceArray(self.ctx, (s.shape[0],))
        self.ctx.lib.prb_critic_value(self.h, ds.ptr, s.shape[0], out.ptr)
        return out.numpy()

    def __del__(self):
        if sys.is_finalizing():  # interpreter teardown: arbitrary order (a context may already be gone)
            return
        try:
            if self.h:
                self.ctx.lib.prb_agent_destroy(self.h)
        except Exception:
            pass


@dataclass
class PpoConfig:  # ppo.hpp:18-27
    gamma: float = 0.99
    gae_lambda: float = 0.95
    clip_eps: float = 0.2
    entropy_coef: float = 0.01
    value_coef: float = 0.5
    epochs_per_update: int = 4
    minibatch_size: int = 1024
    buffer_size: int = 4096
    learning_rate: float = 1e-3

    def c(self):
        return _PpoConfigC(self.gamma, self.gae_lambda, self.clip_eps, self.entropy_coef, self.value_coef,
                           self.epochs_per_update, self.minibatch_size, self.buffer_size, self.learning_rate)


@dataclass
class PpoUpdateStats:  # ppo.hpp:198-203
    mean_policy_loss: float = 0.0
    mean_value_loss: float = 0.0
    mean_entropy: float = 0.0
    minibatches: int = 0


class Rollout:
    """Device TransitionBuffer sized N*H for one VecEnv (buffer.hpp:27-135)."""

    def __init__(self, ctx: Context, handle, N: int, H: int, S: int, A: int, keepalive=None):
        self.ctx, self.h, self.N, self.H, self.S, self.A = ctx, handle, N, H, S, A
        self._keep = keepalive

    @classmethod
    def for_env(cls, env: VectorizedEnvironment, horizon: int) -> "Rollout":
        h = C.c_void_p()
        env.ctx.lib.prb_rollout_create(env.h, horizon, C.byref(h))
        return cls(env.ctx, h, env.num_envs(), horizon, env.state_dim, env.action_dim, keepalive=env)

    @classmethod
    def raw(cls, ctx: Context, N: int, H: int, S: int, A: int) -> "Rollout":
        h = C.c_void_p()
        ctx.lib.prb_rollout_create_raw(ctx.h, N, H, S, A, C.byref(h))
        return cls(ctx, h, N, H, S, A)

    @property
    def capacity(self) -> int:
        return self.N * self.H

    def set_mode(self, mode):
        """2 (default): fused kernel with tcgen05 layers; 1: fused fp32 SIMT; 0: per-step kernels.
        (bools map True -> 1, False -> 0)."""
        self.ctx.lib.prb_rollout_set_mode(self.h, int(mode))

    def collect(self, agent: Agent, env: VectorizedEnvironment, seed: int):
        """worker_collect pod.hpp:95-132."""
        self.ctx.lib.prb_rollout_collect(self.h, agent.h, env.h, seed)

    def download(self):
        n, S, A = self.capacity, self.S, self.A
        out = dict(states=np.zeros((n, S)), actions=np.zeros((n, A)), log_probs=np.zeros(n), rewards=np.zeros(n),
                   dones=np.zeros(n, dtype=np.uint8), values=np.zeros(n), bootstrap=np.zeros(self.N))
        self.ctx.lib.prb_rollout_download(self.h, *[_p(out[k], C.c_uint8 if k == "dones" else C.c_double)
                                                    for k in ("states", "actions", "log_probs", "rewards", "dones",
                                                              "values", "bootstrap")])
        return out

    def download_chunks(self, envs, advantages: bool = False):
        """The chunks of the selected envs only (rows e*H..e*H+H-1 of each env e, pod.hpp:89-94),
        in the order given; raw (un-normalised) GAE advantages/returns when `advantages`."""
        envs = np.ascontiguousarray(envs, dtype=np.uint64)
        n, S, A = envs.size * self.H, self.S, self.A
        out = dict(states=np.zeros((n, S)), actions=np.zeros((n, A)), log_probs=np.zeros(n), rewards=np.zeros(n),
                   dones=np.zeros(n, dtype=np.uint8), values=np.zeros(n), bootstrap=np.zeros(envs.size))
        if advantages:
            out.update(raw_advantages=np.zeros(n), returns=np.zeros(n))
        keys = ("states", "actions", "log_probs", "rewards", "dones", "values", "bootstrap", "raw_advantages",
                "returns")
        self.ctx.lib.prb_rollout_download_chunks(
            self.h, _p(envs, C.c_uint64), envs.size,
            *[_p(out[k], C.c_uint8 if k == "dones" else C.c_double) if k in out else None for k in keys])
        return out

    def gae_stats(self):
        """(mean, denom) of the last buffer_advantages normalisation (ppo.hpp:234-242)."""
        m, d = C.c_double(), C.c_double()
        self.ctx.lib.prb_gae_stats(self.h, C.byref(m), C.byref(d))
        return m.value, d.value

    def upload(self, states, actions, log_probs, rewards, dones, values, bootstrap):
        arrs = [np.ascontiguousarray(x, dtype=np.float64) for x in (states, actions, log_probs, rewards)]
        d = np.ascontiguousarray(dones, dtype=np.uint8)
        v = np.ascontiguousarray(values, dtype=np.float64)
        b = np.ascontiguousarray(bootstrap, dtype=np.float64)
        self.ctx.lib.prb_rollout_upload(self.h, *[_p(a, C.c_double) for a in arrs], _p(d, C.c_uint8),
                                        _p(v, C.c_double), _p(b, C.c_double))

    def buffer_advantages(self, cfg: PpoConfig, normalize: bool = True):
        """buffer_advantages ppo.hpp:212-244 -> (advantages, returns) in reference order."""
        self.ctx.lib.prb_gae(self.h, cfg.gamma, cfg.gae_lambda, 1 if normalize else 0)
        adv, ret = np.zeros(self.capacity), np.zeros(self.capacity)
        self.ctx.lib.prb_gae_download(self.h, _p(adv, C.c_double), _p(ret, C.c_double))
        return adv, ret

    def set_advantages(self, advantages, returns):
        """Seam: gather_minibatch inputs (already-normalised advantages, returns)."""
        a = np.ascontiguousarray(advantages, dtype=np.float64)
        r = np.ascontiguousarray(returns, dtype=np.float64)
        self.ctx.lib.prb_rollout_set_advantages(self.h, _p(a, C.c_double), _p(r, C.c_double))

    def ppo_loss_grads(self, agent: Agent, rows, cfg: PpoConfig):
        rows = np.ascontiguousarray(rows, dtype=np.uint64)
        g = np.zeros(agent.param_count)
        losses = np.zeros(3)
        c = cfg.c()
        self.ctx.lib.prb_ppo_loss_grads(agent.h, self.h, _p(rows, C.c_uint64), rows.size, C.byref(c),
                                        _p(g, C.c_double), _p(losses, C.c_double))
        return losses, g

    def __del__(self):
        if sys.is_finalizing():  # interpreter teardown: arbitrary order (a context may already be gone)
            return
        try:
            if self.h:
                self.ctx.lib.prb_rollout_destroy(self.h)
        except Exception:
            pass


def ppo_update(agent: Agent, rollout: Rollout, cfg: PpoConfig, seed: int, perm: Optional[np.ndarray] = None,
               out: Optional[Agent] = None):
    """ppo_update ppo.hpp:249-296.  Returns (trained copy, PpoUpdateStats); the
    input agent is untouched.  ``perm`` = epochs*n indices in the reference
    index space (e.g. the exact std::shuffle sequence) or None for device
    permutations keyed by ``seed``."""
    dst = out if out is not None else Agent(agent.ctx, agent.state_dim, agent.action_dim, agent.hidden)
    c = cfg.c()
    st = _PpoStatsC()
    pp = None
    if perm is not None:
        perm = np.ascontiguousarray(perm, dtype=np.uint64)
        pp = _p(perm, C.c_uint64)
    agent.ctx.lib.prb_ppo_update(agent.h, rollout.h, C.byref(c), seed, pp, dst.h, C.byref(st))
    return dst, PpoUpdateStats(st.mean_policy_loss, st.mean_value_loss, st.mean_entropy, st.minibatches)


def collect_pods(rollouts: Sequence["Rollout"], agents: Sequence[Agent], envs: Sequence["VectorizedEnvironment"],
                 seeds: Sequence[int]) -> None:
    """worker_collect (pod.hpp:95-132) of every pod in ONE tcgen05 launch (per-pod weights) when all
    pods are stock VecEnvs of the tcgen05 shapes; other pods are collected one by one."""
    P = len(rollouts)
    rs = (C.c_void_p * P)(*[r.h for r in rollouts])
    ag = (C.c_void_p * P)(*[a.h for a in agents])
    es = (C.c_void_p * P)(*[e.h for e in envs])
    sd = np.ascontiguousarray(seeds, dtype=np.uint64)
    agents[0].ctx.lib.prb_rollout_collect_pods(rs, ag, es, P, _p(sd, C.c_uint64))


def ppo_update_learners(agents: Sequence[Agent], rollouts: Sequence[Rollout], cfg: PpoConfig, seeds: Sequence[int],
                        outs: Optional[Sequence[Agent]] = None):
    """pod_train's learner phase (pod.hpp:436-461): learner l = ppo_update(agents[l], rollouts[l],
    cfg, seeds[l]), every learner in ONE tensor-core launch (8 co-resident CTAs each); nets the
    tensor-core update does not support run one after another on the SIMT path.
    Returns (trained copies, [PpoUpdateStats])."""
    L = len(agents)
    dsts = list(outs) if outs is not None else [Agent(a.ctx, a.state_dim, a.action_dim, a.hidden) for a in agents]
    c = cfg.c()
    st = (_PpoStatsC * L)()
    srcs = (C.c_void_p * L)(*[a.h for a in agents])
    ros = (C.c_void_p * L)(*[r.h for r in rollouts])
    dh = (C.c_void_p * L)(*[d.h for d in dsts])
    sd = np.ascontiguousarray(seeds, dtype=np.uint64)
    agents[0].ctx.lib.prb_ppo_update_learners(srcs, ros, L, C.byref(c), _p(sd, C.c_uint64), dh, st)
    return dsts, [PpoUpdateStats(x.mean_policy_loss, x.mean_value_loss, x.mean_entropy, x.minibatches) for x in st]


def fuse_parameters(agents: Sequence[Agent], out: Optional[Agent] = None) -> Agent:
    """fuse_parameters pod.hpp:141-172."""
    if not agents:
        raise UsageError("fuse_parameters: empty artifact list")
    a0 = agents[0]
    dst = out if out is not None else Agent(a0.ctx, a0.state_dim, a0.action_dim, a0.hidden)
    arr = (C.c_void_p * len(agents))(*[a.h.value for a in agents])
    a0.ctx.lib.prb_fuse_parameters(arr, len(agents), dst.h)
    return dst


@dataclass
class EvaluationRecord:
    """EvaluationRecord pod.hpp:30-36 (wall_seconds / env_steps are the caller's)."""
    episodic_rewards: np.ndarray
    mean: float
    std_dev: float
    eval_steps: int


def evaluate(agent: Agent, env: "VectorizedEnvironment", seed: int, sample_actions: bool = False) -> EvaluationRecord:
    """evaluate pod.hpp:43-83: one evaluation episode per env of `env` (which is
    reset with derive_seed(seed, kEpisode, i) and consumed)."""
    n = env.num_envs()
    r = np.zeros(n, dtype=np.float64)
    m, sd, st = C.c_double(), C.c_double(), C.c_uint64()
    agent.ctx.lib.prb_evaluate(agent.h, env.h, seed, 1 if sample_actions else 0, _p(r, C.c_double), C.byref(m),
                               C.byref(sd), C.byref(st))
    return EvaluationRecord(r, m.value, sd.value, st.value)


def evaluate_pods(agents: Sequence[Agent], envs: Sequence["VectorizedEnvironment"], seeds: Sequence[int],
                  sample_actions: bool = False) -> List[EvaluationRecord]:
    """evaluate (pod.hpp:43-83) for every pod of a GPU in one pass: record p equals
    evaluate(agents[p], envs[p], seeds[p]) exactly (one policy launch per step for all pods)."""
    P = len(agents)
    if P == 0:
        return []
    n = envs[0].num_envs()
    r = np.zeros((P, n), dtype=np.float64)
    m, sd, st = np.zeros(P), np.zeros(P), np.zeros(P, dtype=np.uint64)
    ah = (C.c_void_p * P)(*[a.h.value if hasattr(a.h, "value") else a.h for a in agents])
    eh = (C.c_void_p * P)(*[e.h.value if hasattr(e.h, "value") else e.h for e in envs])
    sd_ = np.ascontiguousarray(seeds, dtype=np.uint64)
    agents[0].ctx.lib.prb_evaluate_pods(ah, eh, P, _p(sd_, C.c_uint64), 1 if sample_actions else 0,
                                        _p(r, C.c_double), _p(m, C.c_double), _p(sd, C.c_double),
                                        _p(st, C.c_uint64))
    return [EvaluationRecord(r[p], float(m[p]), float(sd[p]), int(st[p])) for p in range(P)]


def leaderboard_rank(ctx: Context, scores, seqs, capacity: int) -> np.ndarray:
    """Board order after inserting (score, seq) candidates (tournament.hpp:104-119)."""
    s = np.ascontiguousarray(scores, dtype=np.float64)
    q = np.ascontiguousarray(seqs, dtype=np.uint64)
    order = np.zeros(max(capacity, 1), dtype=np.int32)
    cnt = C.c_int32()
    ctx.lib.prb_leaderboard_rank_host(ctx.h, _p(s, C.c_double), _p(q, C.c_uint64), s.size, capacity,
                                      _p(order, C.c_int32), C.byref(cnt))
    return order[:cnt.value]


class PopulationStats:  # tournament.hpp:38-41
    def __init__(self, mean: np.ndarray, variance: np.ndarray):
        self.mean, self.variance = mean, variance


def leaderboard_stats(entries: Sequence[Agent]) -> PopulationStats:
    """Leaderboard::refresh_stats (tournament.hpp:66-87) over the board's entries in board order:
    per-coordinate mean and population variance of the flat params, computed on the device."""
    if not entries:
        return PopulationStats(np.zeros(0), np.zeros(0))
    P = entries[0].param_count
    arr = (C.c_void_p * len(entries))(*[e.h for e in entries])
    mean, var = np.zeros(P), np.zeros(P)
    entries[0].ctx.lib.prb_leaderboard_stats_host(arr, len(entries), _p(mean, C.c_double), _p(var, C.c_double))
    return PopulationStats(mean, var)


def set_debug_option(option: int, value: int) -> None:
    """Test-only switches (PRB_OPT_* in include/prb.h)."""
    _lib.lib().prb_debug_set_option(option, value)


OPT_PPO_PER_KERNEL, OPT_TC_FORCE_REDO, OPT_PM_CTA_PAIR = 1, 2, 3


@dataclass
class CheckpointInfo:  # lineage, algo_tag and CheckpointMeta of a PODRCKPT file (checkpoint.hpp:200-205)
    parent_pod: int = -1
    mutation_seed: int = 0
    algo_tag: str = "ppo"
    meta: Optional[tuple] = None


def checkpoint_encode(agent: Agent, info: CheckpointInfo = CheckpointInfo()) -> bytes:
    """encode_checkpoint(artifact_to_tensors(agent)) -- PODRCKPT v1 bytes (checkpoint.hpp:122-245)."""
    meta = np.ascontiguousarray(info.meta, dtype=np.float64) if info.meta is not None else None
    size = C.c_size_t()
    args = (agent.h, info.parent_pod, info.mutation_seed, info.algo_tag.encode(),
            _p(meta, C.c_double) if meta is not None else None)
    agent.ctx.lib.prb_checkpoint_encode(*args, None, 0, C.byref(size))
    out = np.zeros(size.value, dtype=np.uint8)
    agent.ctx.lib.prb_checkpoint_encode(*args, _p(out, C.c_uint8), out.size, C.byref(size))
    return out.tobytes()


def checkpoint_decode(agent: Agent, data: bytes) -> CheckpointInfo:
    """decode_checkpoint + artifact_from_tensors into `agent` (checkpoint.hpp:145-303)."""
    b = np.frombuffer(data, dtype=np.uint8).copy()
    parent, seed, has = C.c_int64(), C.c_uint64(), C.c_int()
    tag = C.create_string_buffer(256)
    meta = np.zeros(3)
    agent.ctx.lib.prb_checkpoint_decode(agent.h, _p(b, C.c_uint8), b.size, C.byref(parent), C.byref(seed), tag, 256,
                                        _p(meta, C.c_double), C.byref(has))
    return CheckpointInfo(parent.value, seed.value, tag.value.decode(), tuple(meta) if has.value else None)


def save_checkpoint(agent: Agent, path: str, info: CheckpointInfo = CheckpointInfo()) -> None:
    meta = np.ascontiguousarray(info.meta, dtype=np.float64) if info.meta is not None else None
    agent.ctx.lib.prb_checkpoint_save(agent.h, path.encode(), info.parent_pod, info.mutation_seed,
                                      info.algo_tag.encode(), _p(meta, C.c_double) if meta is not None else None)


def load_checkpoint(agent: Agent, path: str) -> CheckpointInfo:
    parent, seed, has = C.c_int64(), C.c_uint64(), C.c_int()
    tag = C.create_string_buffer(256)
    meta = np.zeros(3)
    agent.ctx.lib.prb_checkpoint_load(agent.h, path.encode(), C.byref(parent), C.byref(seed), tag, 256,
                                      _p(meta, C.c_double), C.byref(has))
    return CheckpointInfo(parent.value, seed.value, tag.value.decode(), tuple(meta) if has.value else None)
