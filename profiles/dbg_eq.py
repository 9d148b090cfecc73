"""Bit-equality check of the persistent PPO update's A/B knobs against the per-kernel path
(PRB_PPO_GRAPH=1) at a configs[0]-like shape: prints, per knob, how many params / m / v differ.
    python profiles/dbg_eq.py"""
import os, sys, numpy as np
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
from paper_2112_05923_b200 import podracer as pr
from test_gpu_learn import _upload_random_buffer
ctx = pr.Context(0)
S, A, hid, N, H, mb, epochs = 181, 30, (64, 64), 64, 64, 1024, 2
for trial in range(3):
    rng = np.random.default_rng(S + mb)
    agent = pr.Agent.init(ctx, S, A, seed=3, hidden=hid)
    ro, _ = _upload_random_buffer(pr, ctx, rng, N, H, S, A)
    cfg = pr.PpoConfig(epochs_per_update=epochs, minibatch_size=mb, buffer_size=N * H)
    res = {}
    for mode in ("spec", "nospec", "cpasync", "graph"):
        for k in ("PRB_PPO_NOSPEC", "PRB_PPO_CPASYNC", "PRB_PPO_GRAPH"): os.environ.pop(k, None)
        if mode == "nospec": os.environ["PRB_PPO_NOSPEC"] = "1"
        if mode == "cpasync": os.environ["PRB_PPO_CPASYNC"] = "1"
        if mode == "graph": os.environ["PRB_PPO_GRAPH"] = "1"
        a1, s1 = pr.ppo_update(agent, ro, cfg, 21)
        res[mode] = a1.get()
    for mode in ("spec", "nospec", "cpasync"):
        for nm, x, y in zip("pmv", res[mode][:3], res["graph"][:3]):
            d = np.nonzero(x != y)[0]
            print(trial, mode, nm, len(d), d[:8], (np.abs(x - y).max() if len(d) else 0))
        print(trial, mode, "t", res[mode][3], res["graph"][3])
