#!/usr/bin/env python
"""Device time of one PPO update at the configs[0] shape (1,024 stock envs x 256 steps, 4 epochs x
256 minibatches of 1,024 rows): the tensor-core cluster update (mode 1) vs the fp32 SIMT
persistent update (mode 0), CUDA events around the update kernel (prb_ctx_profile, PPO class)."""
import ctypes as C
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2112_05923_b200 import podracer as pr  # noqa: E402

K, S = 30, 181
N = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
EP = int(sys.argv[2]) if len(sys.argv) > 2 else 4
ctx = pr.Context(0)
m = pr.synthetic_market(K, 2048, 2112)
ind = pr.compute_indicators(m["high"], m["low"], m["close"])
market = pr.MarketData(ctx, m["close"], ind)
env = pr.VectorizedEnvironment.stock(ctx, market, pr.StockConfig(), 0, 2047, N)
env.reset(3)
agent = pr.Agent.init(ctx, S, K, seed=7)
ro = pr.Rollout.for_env(env, 256)
ro.collect(agent, env, seed=5)
cfg = pr.PpoConfig(epochs_per_update=EP, minibatch_size=1024, buffer_size=N * 256)
for mode in (1, 0):
    agent.set_ppo_mode(mode)
    out = pr.Agent(ctx, S, K)
    pr.ppo_update(agent, ro, cfg, 11, out=out)  # warm (workspace)
    ctx.synchronize()
    ctx.lib.prb_ctx_profile(ctx.h, 1)
    reps = 3
    for r in range(reps):
        _, st = pr.ppo_update(agent, ro, cfg, 11 + r, out=out)
    ctx.synchronize()
    tot = 0.0
    for kind in (4, 5, 6):
        ms, n = C.c_double(), C.c_uint64()
        ctx.lib.prb_ctx_profile_read(ctx.h, kind, C.byref(ms), C.byref(n))
        tot += ms.value
    ctx.lib.prb_ctx_profile(ctx.h, 0)
    print(json.dumps({"mode": mode, "envs": N, "epochs": EP, "update_ms": tot / reps,
                      "us_per_minibatch": tot / reps * 1e3 / st.minibatches, "minibatches": st.minibatches,
                      "policy_loss": st.mean_policy_loss, "value_loss": st.mean_value_loss}), flush=True)
