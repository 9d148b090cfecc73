#!/usr/bin/env python
"""Stage times of one configs[3] generation (8 pods x 1,024 envs x 256, 2 learners each) on one
GPU: the PodPopulation.generation() stages, each bracketed by a device synchronisation."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2112_05923_b200 import podracer as pr  # noqa: E402
from paper_2112_05923_b200 import tournament as tn  # noqa: E402

ctx = pr.Context(0)
m, ind = bench.market_arrays()
market = pr.MarketData(ctx, m["close"], ind)
N, H, P, L = 1024, 256, 8, 2
pcfg = pr.PpoConfig(minibatch_size=1024, epochs_per_update=4, buffer_size=N * H)
pop = tn.PodPopulation(ctx, market, pr.StockConfig(), pods=P, envs_per_pod=N, horizon=H, learners=L, ppo_cfg=pcfg,
                       window=(0, bench.T_ROWS - 1), eval_episodes=10, eval_window=(1900, 1940), capacity=10,
                       top_k=3, seed=2112)
pop.generation()
T = {}


def tick(name, t0):
    ctx.synchronize()
    T[name] = T.get(name, 0.0) + (time.perf_counter() - t0) * 1e3
    return time.perf_counter()


for g in range(3):
    t = time.perf_counter()
    pr.collect_pods(pop.rollouts, pop.agents, pop.envs, [pr.derive_seed(1, 2, p, g) for p in range(P)])
    t = tick("collect", t)
    srcs = [a for a in pop.agents for _ in range(L)]
    ros = [r for r in pop.rollouts for _ in range(L)]
    outs = [o for lo in pop.learner_out for o in lo]
    pr.ppo_update_learners(srcs, ros, pcfg, list(range(len(srcs))), outs=outs)
    t = tick("learners", t)
    for p in range(P):
        pr.fuse_parameters(pop.learner_out[p], out=pop.agents[p])
    t = tick("fuse", t)
    scores = np.array([r.mean for r in pr.evaluate_pods(pop.agents, pop.eval_envs, [7 + p for p in range(P)])])
    t = tick("evaluate", t)
    order = pr.leaderboard_rank(ctx, scores, np.arange(P, dtype=np.uint64), 10)
    t = tick("rank", t)
    for j in range(3):
        pop.elites[j].copy_from(pop.agents[int(order[j])])
    for p in range(3):
        pop.agents[p].init_device(11 + p)
    for p in range(3, P):
        pop.agents[p].copy_from(pop.elites[p % 3])
        pop.agents[p].mutate(13 + p, 0.02)
    t = tick("select+init+mutate", t)
print({k: round(v / 3, 2) for k, v in T.items()}, "ms per generation")
