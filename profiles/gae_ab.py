#!/usr/bin/env python
"""GAE kernel A/B: average gae_scan_kernel time on a collected configs[1] buffer (65,536 envs x
256 steps), 17 algorithmic bytes per transition (read r, V, done; write adv, ret).
Run once per build: PRB_LIB_PATH=profiles/ab/libprb_<v>.so python profiles/gae_ab.py"""
import ctypes as C
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2112_05923_b200 import podracer as pr  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 65536
H = int(sys.argv[2]) if len(sys.argv) > 2 else 256
ctx = pr.Context(0)
m = pr.synthetic_market(30, 2048, 2112)
ind = pr.compute_indicators(m["high"], m["low"], m["close"])
market = pr.MarketData(ctx, m["close"], ind)
env = pr.VectorizedEnvironment.stock(ctx, market, pr.StockConfig(), 1900, 2047, N)
env.reset(1)
agent = pr.Agent.init(ctx, 181, 30, seed=7)
ro = pr.Rollout.for_env(env, H)
ro.collect(agent, env, seed=1)
for _ in range(3):
    ctx.lib.prb_gae(ro.h, 0.99, 0.95, 1)
ctx.synchronize()
ctx.lib.prb_ctx_profile(ctx.h, 1)
for _ in range(30):
    ctx.lib.prb_gae(ro.h, 0.99, 0.95, 1)
ctx.synchronize()
ms, n = C.c_double(), C.c_uint64()
ctx.lib.prb_ctx_profile_read(ctx.h, 3, C.byref(ms), C.byref(n))
us = ms.value / n.value * 1e3
gbs = N * H * 17 / (us * 1e-6) / 1e9
print(json.dumps({"lib": os.environ.get("PRB_LIB_PATH", "default"), "N": N, "H": H, "kernel_us": us, "gbs": gbs,
                  "frac_hbm": gbs / 6548.5, "stats": ro.gae_stats()}))
