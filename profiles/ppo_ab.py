"""A/B of a persistent PPO update knob at configs[0] (1,024 stock envs x 256, minibatch 1,024,
4 epochs = 1,024 Adam steps): the default build vs the same with VAR=1 -- PRB_PPO_CPASYNC
(per-thread cp.async weight staging instead of bulk copies of the staged-layout image, the
default VAR) or PRB_PPO_NOSPEC (Adam stored after the gate barrier instead of speculatively
before it). Device-timed with CUDA events; also checks both give bit-identical parameters.
    python profiles/ppo_ab.py [VAR]"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2112_05923_b200 import podracer as pr  # noqa: E402

ctx = pr.Context(0)
m, ind = bench.market_arrays()
market = pr.MarketData(ctx, m["close"], ind)
N, H = 1024, 256
env = pr.VectorizedEnvironment.stock(ctx, market, pr.StockConfig(), 0, bench.T_ROWS - 1, N)
env.reset(3)
agent = pr.Agent.init(ctx, bench.S_DIM, bench.K_ASSETS, seed=7)
ro = pr.Rollout.for_env(env, H)
ro.collect(agent, env, seed=1)
cfg = pr.PpoConfig(minibatch_size=1024, epochs_per_update=4, buffer_size=N * H)
VAR = sys.argv[1] if len(sys.argv) > 1 else "PRB_PPO_CPASYNC"
outs = {}
for name, flag in (("default", None), (VAR, "1")) * 4:
    if flag:
        os.environ[VAR] = flag
    else:
        os.environ.pop(VAR, None)
    out = pr.Agent.init(ctx, bench.S_DIM, bench.K_ASSETS, seed=7)
    pr.ppo_update(agent, ro, cfg, seed=2, out=out)  # warm
    ts = []
    for _ in range(5):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        s.record()
        pr.ppo_update(agent, ro, cfg, seed=2, out=out)
        e.record()
        torch.cuda.synchronize()
        ts.append(s.elapsed_time(e))
    outs[name] = out.flatten_params()
    print(f"{name:16s} update {np.median(ts):7.2f} ms = {np.median(ts) / 1024 * 1e3:6.2f} us/minibatch (min {min(ts):.2f})")
print("bit-identical params:", np.array_equal(outs["default"], outs[VAR]))
