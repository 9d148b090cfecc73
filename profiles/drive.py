#!/usr/bin/env python
"""Small deterministic drivers for ncu captures (one kernel family each).

  python profiles/drive.py collect  [N] [H]   # fused stock rollout (or --unfused)
  python profiles/drive.py env      [N]       # prb_vecenv_step on device buffers
  python profiles/drive.py ppo      [N] [H]   # a few PPO minibatch steps (--tc: tensor-core path)
  python profiles/drive.py learners [L] [N]   # L concurrent tensor-core learners (one cluster each)
  python profiles/drive.py pm       [N] [H]   # PointMass 3x256 tcgen05 rollout (configs[2])
  python profiles/drive.py gae      [N] [H]   # buffer_advantages on a collected configs[1] buffer
  python profiles/drive.py adam     [P]       # adam_step on a 10.5M-param agent (> L2)
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2112_05923_b200 import podracer as pr  # noqa: E402


def setup(N):
    ctx = pr.Context(0)
    m = pr.synthetic_market(30, 2048, 2112)
    ind = pr.compute_indicators(m["high"], m["low"], m["close"])
    market = pr.MarketData(ctx, m["close"], ind)
    env = pr.VectorizedEnvironment.stock(ctx, market, pr.StockConfig(), 0, 2047, N)
    env.reset(1)
    return ctx, market, env


def main():
    what = sys.argv[1]
    fused = "--unfused" not in sys.argv
    args = [a for a in sys.argv[2:] if not a.startswith("--")]
    if what == "collect":
        N = int(args[0]) if args else 65536
        H = int(args[1]) if len(args) > 1 else 32
        ctx, market, env = setup(N)
        agent = pr.Agent.init(ctx, 181, 30, seed=7)
        ro = pr.Rollout.for_env(env, H)
        ro.set_mode(1 if "--simt" in sys.argv else (2 if fused else 0))
        for i in range(3):
            ro.collect(agent, env, seed=i)
        ctx.synchronize()
    elif what == "env":
        N = int(args[0]) if args else 1 << 20
        ctx, market, env = setup(N)
        a = pr.DeviceArray.from_numpy(ctx, np.random.default_rng(0).uniform(-1.2, 1.2, (N, 30)).astype(np.float32))
        r, d = ctx.alloc((N,)), ctx.alloc((N,), np.uint8)
        for _ in range(6):
            env.step_device(a.ptr, r.ptr, d.ptr)
        ctx.synchronize()
    elif what == "ppo":
        N = int(args[0]) if args else 4096
        H = int(args[1]) if len(args) > 1 else 64
        ctx, market, env = setup(N)
        agent = pr.Agent.init(ctx, 181, 30, seed=7)
        ro = pr.Rollout.for_env(env, H)
        ro.collect(agent, env, seed=1)
        cfg = pr.PpoConfig(minibatch_size=1024, epochs_per_update=1, buffer_size=N * H)
        agent.set_ppo_mode(1 if "--tc" in sys.argv else 0)
        pr.ppo_update(agent, ro, cfg, seed=3)
        ctx.synchronize()
    elif what == "learners":
        L = int(args[0]) if args else 16
        N = int(args[1]) if len(args) > 1 else 1024
        H = 64
        ctx, market, env = setup(N)
        agent = pr.Agent.init(ctx, 181, 30, seed=7)
        agent.set_ppo_mode(1)
        ro = pr.Rollout.for_env(env, H)
        ro.collect(agent, env, seed=1)
        cfg = pr.PpoConfig(minibatch_size=1024, epochs_per_update=1, buffer_size=N * H)
        pr.ppo_update_learners([agent] * L, [ro] * L, cfg, list(range(L)))
        ctx.synchronize()
    elif what == "pm":
        N = int(args[0]) if args else 262144
        H = int(args[1]) if len(args) > 1 else 16
        ctx = pr.Context(0)
        env = pr.VectorizedEnvironment.pointmass(ctx, N)
        env.reset(7)
        agent = pr.Agent.init(ctx, 6, 2, seed=7, hidden=(256, 256, 256))
        ro = pr.Rollout.for_env(env, H)
        for i in range(2):
            ro.collect(agent, env, seed=i)
        ctx.synchronize()
    elif what == "gae":
        N = int(args[0]) if args else 65536
        H = int(args[1]) if len(args) > 1 else 256
        ctx, market, env = setup(N)
        agent = pr.Agent.init(ctx, 181, 30, seed=7)
        ro = pr.Rollout.for_env(env, H)
        ro.collect(agent, env, seed=1)
        for _ in range(3):
            ctx.lib.prb_gae(ro.h, 0.99, 0.95, 1)
        ctx.synchronize()
    elif what == "adam":
        import ctypes as C
        ctx = pr.Context(0)
        agent = pr.Agent.init(ctx, 4096, 2, seed=1, hidden=(1024, 1024))
        g = pr.DeviceArray.from_numpy(ctx, np.random.default_rng(0).normal(size=agent.param_count).astype(np.float32)
                                      * 1e-3)
        for _ in range(3):
            ctx.lib.prb_adam_step_device(agent.h, C.c_void_p(g.ptr))
        ctx.synchronize()
    print("ok", what)


if __name__ == "__main__":
    main()
