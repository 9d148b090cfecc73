"""Where the time of one configs[0] PPO iteration goes on the GPU (not a bench line):
collect (1,024 stock envs x 256) and ppo_update (GAE + 4 epochs x 256 minibatches of
1,024 + Adam), each timed with CUDA events on the context stream and with the host
wall clock around the call.   python profiles/c1_breakdown.py"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2112_05923_b200 import podracer as pr  # noqa: E402

lib = pr._lib.lib()
ctx = pr.Context(0)
m, ind = bench.market_arrays()
market = pr.MarketData(ctx, m["close"], ind)
cfg = pr.StockConfig()
N, H = int(os.environ.get("C1_N", 1024)), 256
env = pr.VectorizedEnvironment.stock(ctx, market, cfg, 0, bench.T_ROWS - 1, N)
env.reset(3)
agent = pr.Agent.init(ctx, bench.S_DIM, bench.K_ASSETS, seed=7)
ro = pr.Rollout.for_env(env, H)
pcfg = pr.PpoConfig(minibatch_size=1024, epochs_per_update=4, buffer_size=N * H)
for i in range(2):
    ro.collect(agent, env, seed=100 + i)
    pr.ppo_update(agent, ro, pcfg, seed=200 + i, out=agent)
ctx.synchronize()
for i in range(3):
    t0 = time.perf_counter()
    c_ms = bench.time_region(lib, ctx, lambda: ro.collect(agent, env, seed=300 + i))
    t1 = time.perf_counter()
    u_ms = bench.time_region(lib, ctx, lambda: pr.ppo_update(agent, ro, pcfg, seed=400 + i, out=agent))
    t2 = time.perf_counter()
    print(f"N={N}: collect dev {c_ms:.2f} ms host {1e3 * (t1 - t0):.2f} ms | ppo_update dev {u_ms:.2f} ms "
          f"host {1e3 * (t2 - t1):.2f} ms ({u_ms * 1e3 / (4 * N * H // 1024):.1f} us/minibatch)", flush=True)
