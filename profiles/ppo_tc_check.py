#!/usr/bin/env python
"""Development check of the tensor-core PPO update (ppo_tc.cu): one minibatch step at lr = 0 on a
real collected stock buffer, the device's reduced gradient (prb_debug_agent_grads) against
orc_ppo_loss_grads on the same rows (the injected permutation), per parameter block; then a
multi-step update against the SIMT path."""
import ctypes as C
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from oracle_bind import PpoCfg, load_oracle, ptr, SZ, U8, U64  # noqa: E402
from paper_2112_05923_b200 import podracer as pr  # noqa: E402

K, S = 30, 181
orc = load_oracle()
ctx = pr.Context(0)
m = pr.synthetic_market(K, 2048, 2112)
ind = pr.compute_indicators(m["high"], m["low"], m["close"])
market = pr.MarketData(ctx, m["close"], ind)
mb = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
N, H = 64, 64
n = N * H
env = pr.VectorizedEnvironment.stock(ctx, market, pr.StockConfig(), 1500, 2047, N)
env.reset(5)
agent = pr.Agent.init(ctx, S, K, seed=7)
ro = pr.Rollout.for_env(env, H)
ro.collect(agent, env, seed=77)
buf = ro.download()
rng = np.random.default_rng(1)
perm = rng.permutation(n).astype(np.uint64)
cfg = pr.PpoConfig(epochs_per_update=1, minibatch_size=mb, buffer_size=n, learning_rate=0.0)
# one step: buffer n but only the first minibatch matters -> use an update of exactly 1 step
CLIP = float(sys.argv[2]) if len(sys.argv) > 2 else 0.2
cfg1 = pr.PpoConfig(epochs_per_update=1, minibatch_size=mb, buffer_size=n, learning_rate=0.0, clip_eps=CLIP)
out = pr.Agent(ctx, S, K)
try:
    new, st = pr.ppo_update(agent, ro, cfg1, 3, perm=perm, out=out)
except pr.NumericError as ex:
    print("NumericError", ex, "accepted steps", out.get()[3])
    st = None
g = np.zeros(agent.param_count)
ctx.lib.prb_debug_agent_grads(out.h, g.ctypes.data_as(C.POINTER(C.c_double)))
print("non-finite grads:", int(np.sum(~np.isfinite(g))), "first idx", np.where(~np.isfinite(g))[0][:20])
# the last step's rows are perm[(nmb-1)*mb : nmb*mb]
nmb = n // mb
rows = perm[(nmb - 1) * mb: nmb * mb]
adv, ret = ro.buffer_advantages(cfg1, normalize=True)
flat = agent.flatten_params()
og = np.zeros(flat.size); ol = np.zeros(3)
idx = rows.astype(np.int64)
dA = np.array([S, 64, 64, K], dtype=np.uint64); dC = np.array([S, 64, 64, 1], dtype=np.uint64)
oc = PpoCfg(0.99, 0.95, CLIP, 0.01, 0.5, 1, mb, n, 0.0)
st_rows = np.ascontiguousarray(buf["states"][idx]); ac_rows = np.ascontiguousarray(buf["actions"][idx])
rc = orc.orc_ppo_loss_grads(ptr(flat), ptr(dA, SZ), 3, ptr(dC, SZ), 3, ptr(st_rows), ptr(ac_rows),
                            ptr(np.ascontiguousarray(buf["log_probs"][idx])), ptr(np.ascontiguousarray(adv[idx])),
                            ptr(np.ascontiguousarray(ret[idx])), mb, C.byref(oc), ptr(og), ptr(ol))
print("orc rc", rc, "losses", ol, "device stats", st)
# blocks of the flat layout
blocks = []
off = 0
for name, (i, o) in [("a.W1", (S, 64)), ("a.W2", (64, 64)), ("a.W3", (64, K))]:
    blocks += [(name, off, off + i * o), (name.replace("W", "b"), off + i * o, off + i * o + o)]
    off += i * o + o
blocks.append(("log_std", off, off + K)); off += K
for name, (i, o) in [("c.W1", (S, 64)), ("c.W2", (64, 64)), ("c.W3", (64, 1))]:
    blocks += [(name, off, off + i * o), (name.replace("W", "b"), off + i * o, off + i * o + o)]
    off += i * o + o
for name, lo, hi in blocks:
    d, o_ = g[lo:hi], og[lo:hi]
    scale = max(np.max(np.abs(o_)), 1e-30)
    print(json.dumps({"block": name, "max_abs_orc": float(scale), "max_err_rel_to_max": float(np.max(np.abs(d - o_)) / scale),
                      "corr": float(np.corrcoef(d, o_)[0, 1]) if d.size > 1 and np.std(o_) > 0 else None}))

# ---- timing: a configs[0]-shaped update (1,024 envs x 256, 4 epochs x 256 minibatches of 1,024) ----
import time
env2 = pr.VectorizedEnvironment.stock(ctx, market, pr.StockConfig(), 0, 2047, 1024)
env2.reset(3)
ro2 = pr.Rollout.for_env(env2, 256)
ro2.collect(agent, env2, seed=5)
cfgT = pr.PpoConfig(epochs_per_update=4, minibatch_size=1024, buffer_size=1024 * 256)
for mode in (1, 0, 1):
    agent.set_ppo_mode(mode)
    outT = pr.Agent(ctx, S, K)
    pr.ppo_update(agent, ro2, cfgT, 11, out=outT)
    ctx.synchronize()
    t0 = time.perf_counter()
    _, stT = pr.ppo_update(agent, ro2, cfgT, 11, out=outT)
    ctx.synchronize()
    dt = time.perf_counter() - t0
    print(json.dumps({"mode": mode, "update_ms": dt * 1e3, "us_per_minibatch": dt * 1e6 / stT.minibatches,
                      "policy_loss": stT.mean_policy_loss, "value_loss": stT.mean_value_loss,
                      "params_finite": bool(np.all(np.isfinite(outT.flatten_params())))}))
