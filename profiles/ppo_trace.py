"""Phase timeline of one minibatch step of the persistent PPO update (PRB_PPO_TRACE).
Runs one configs[0]-shaped update (1,024 stock envs x 256, minibatch 1,024) with the
trace enabled and prints, for step 4, when the phases end (max over CTAs) relative to
the step start, and how long each grid barrier took to release.
    python profiles/ppo_trace.py"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
path = os.path.join(ROOT, "gpurun_out", "ppo_trace.bin")
os.makedirs(os.path.dirname(path), exist_ok=True)
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
cfg = pr.PpoConfig(minibatch_size=1024, epochs_per_update=1, buffer_size=N * H)
pr.ppo_update(agent, ro, cfg, seed=2)
os.environ["PRB_PPO_TRACE"] = path
pr.ppo_update(agent, ro, cfg, seed=3)
del os.environ["PRB_PPO_TRACE"]
raw = np.fromfile(path, dtype=np.uint64).astype(np.int64)
marks = raw[-32:].reshape(2, 16)
t = raw[:-32].reshape(-1, 16)
t = t[t[:, 0] > 0]
t0 = t[:, 0].min()
names = ["step start", "A done", "barrier 1 exit", "B done", "barrier 2 exit", "C1 done", "barrier 3 exit",
         "C2 (gate+Adam) done", "barrier 4 exit"]
print(f"{len(t)} CTAs; times in us from the earliest step start (min / median / max over CTAs)")
for i, nm in enumerate(names):
    c = (t[:, i] - t0) / 1e3
    print(f"  {nm:22s} {c.min():8.2f} {np.median(c):8.2f} {c.max():8.2f}")
mk_names = ["weights issued", "gather issued", "gather landed", "weights landed", "sync", "layer 0", "layer 1", "layer 2", "inputs stored", "head grads", "head stored",
            "bwd 2->1", "stored", "bwd 1->0", "stored"]  # fwd_delta_r8's marks (3-layer nets)
for net in (0, 1):
    mk = marks[net]
    mk = mk[mk > 0]
    print(["actor", "critic"][net], "row block 0 (SM cycles from block start):",
          ", ".join(f"{n} {int(c - mk[0])}" for n, c in zip(mk_names, mk[1:])))
# phase B per gradient tile (virtual CTA vb = blockIdx.x = tile * RS + split when the grid covers it)
RS = int(os.environ.get("TRACE_RS", "26"))
bdur = (t[:, 3] - t[:, 2]) / 1e3
ntile = (len(bdur) + RS - 1) // RS
bl = (t[:, 10] - t[:, 2]) / 1e3
bc = (t[:, 11] - t[:, 10]) / 1e3
bs = (t[:, 3] - t[:, 11]) / 1e3
ok = t[:, 10] > 0
print("phase B split (us, median/max over CTAs): loads %.2f/%.2f compute %.2f/%.2f stores %.2f/%.2f" % (
    np.median(bl[ok]), bl[ok].max(), np.median(bc[ok]), bc[ok].max(), np.median(bs[ok]), bs[ok].max()))
print("phase B duration per tile (max over its splits, us):",
      " ".join(f"{i}:{bdur[i * RS:(i + 1) * RS].max():.1f}" for i in range(min(ntile, 12))))
adur = (t[:, 1] - t[:, 0]) / 1e3
print("phase A duration: actor CTAs max %.1f us, critic CTAs max %.1f us" % (adur[:128].max(), adur[128:256].max()))
