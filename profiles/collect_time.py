#!/usr/bin/env python
"""Wall time of the stock tcgen05 collect (configs[1] market window, H=256) for several VecEnv
sizes: python profiles/collect_time.py 56832 65536 75776 ...  (synchronised, 5 timed runs)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2112_05923_b200 import podracer as pr  # noqa: E402

ctx = pr.Context(0)
m, ind = bench.market_arrays()
market = pr.MarketData(ctx, m["close"], ind)
H = int(os.environ.get("H", 256))
for N in [int(x) for x in sys.argv[1:]]:
    env = pr.VectorizedEnvironment.stock(ctx, market, pr.StockConfig(), 0, bench.T_ROWS - 1, N)
    env.reset(3)
    agent = pr.Agent.init(ctx, bench.S_DIM, bench.K_ASSETS, seed=7)
    ro = pr.Rollout.for_env(env, H)
    for i in range(2):
        ro.collect(agent, env, seed=i)
    ctx.synchronize()
    ts = []
    for i in range(5):
        t0 = time.perf_counter()
        ro.collect(agent, env, seed=10 + i)
        ctx.synchronize()
        ts.append(time.perf_counter() - t0)
    ms = sorted(ts)[2] * 1e3
    print(f"N={N:8d} ({N / 128 / 148:.2f} tiles/SM): {ms:.3f} ms, {N * H / ms * 1e3:.3e} transitions/s", flush=True)
    del ro, env
