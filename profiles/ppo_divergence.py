#!/usr/bin/env python
"""How the device ppo_update drifts from the f64 oracle with the number of Adam steps at the
headline net (181-64-64-30 / 181-64-64-1, minibatch 1,024) on a real collected buffer, under the
reference's std::shuffle permutation.  For each step count S (buffer = S x 1,024 transitions,
one epoch): max |dp|, the fraction of params off by more than 2e-5 * S, the relative L2 distance
|p_dev - p_orc| / |p_orc - p_0|, and the mean losses.  JSON lines on stdout."""
import ctypes as C
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from oracle_bind import PpoCfg, load_oracle, load_ref, ptr, SZ, U8, U64  # noqa: E402
from paper_2112_05923_b200 import podracer as pr  # noqa: E402

K, S = 30, 181
orc, ref = load_oracle(), load_ref()
ctx = pr.Context(0)
m = pr.synthetic_market(K, 2048, 2112)
ind = pr.compute_indicators(m["high"], m["low"], m["close"])
market = pr.MarketData(ctx, m["close"], ind)
for steps in [int(x) for x in (sys.argv[1:] or ["1", "2", "4", "16", "64"])]:
    H = 256
    N = steps * 1024 // H
    n = N * H
    env = pr.VectorizedEnvironment.stock(ctx, market, pr.StockConfig(), 1500, 2047, N)
    env.reset(5)
    agent = pr.Agent.init(ctx, S, K, seed=7)
    ro = pr.Rollout.for_env(env, H)
    ro.collect(agent, env, seed=77)
    buf = ro.download()
    perms = np.zeros(n, dtype=np.uint64)
    ref.ref_ppo_permutations(4242, n, 1, ptr(perms, U64))
    cfg = pr.PpoConfig(epochs_per_update=1, minibatch_size=1024, buffer_size=n)
    new, st = pr.ppo_update(agent, ro, cfg, 4242, perm=perms)
    p0 = agent.flatten_params()
    fo = p0.copy(); mo = np.zeros(p0.size); vo = np.zeros(p0.size); to = C.c_int64(0); so = np.zeros(4)
    offs = np.arange(N, dtype=np.uint64) * H; lens = np.full(N, H, dtype=np.uint64)
    oc = PpoCfg(0.99, 0.95, 0.2, 0.01, 0.5, 1, 1024, n, 1e-3)
    dA = np.array([S, 64, 64, K], dtype=np.uint64); dC = np.array([S, 64, 64, 1], dtype=np.uint64)
    assert orc.orc_ppo_update(ptr(fo), ptr(mo), ptr(vo), C.byref(to), ptr(dA, SZ), 3, ptr(dC, SZ), 3,
                              ptr(buf["states"]), ptr(buf["actions"]), ptr(buf["log_probs"]), ptr(buf["rewards"]),
                              ptr(buf["dones"], U8), ptr(buf["values"]), n, S, ptr(offs, SZ), ptr(lens, SZ),
                              ptr(buf["bootstrap"]), N, C.byref(oc), ptr(perms, U64), ptr(so)) == 0
    p = new.flatten_params()
    dp = np.abs(p - fo)
    print(json.dumps({"steps": steps, "max_dp": float(dp.max()), "frac_over_2e-5xS": float(np.mean(dp > 2e-5 * steps)),
                      "n_over": int(np.sum(dp > 2e-5 * steps)), "rel_l2": float(np.linalg.norm(p - fo) / np.linalg.norm(fo - p0)),
                      "policy_loss": [st.mean_policy_loss, so[0]], "value_loss": [st.mean_value_loss, so[1]],
                      "entropy": [st.mean_entropy, so[2]]}), flush=True)
