"""GPU (>= 2 devices): NCCL leaderboard all-gather + ranking and elite broadcast
(tests/mgpu_tournament.py under torchrun); two devices driven from two threads of one process.
Skipped on single-GPU boxes."""
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _gpus():
    try:
        out = subprocess.run(["nvidia-smi", "-L"], capture_output=True, text=True, timeout=60).stdout
        return sum(1 for line in out.splitlines() if line.startswith("GPU "))
    except Exception:
        return 0


@pytest.mark.skipif(_gpus() < 2, reason="needs >= 2 GPUs")
def test_tournament_two_ranks():
    n = min(_gpus(), 4)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", "29533", os.path.join(ROOT, "tests", "mgpu_tournament.py")]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0 and "MGPU TOURNAMENT OK" in r.stdout, r.stdout[-3000:] + r.stderr[-3000:]


def _pipeline(pr, dev, out, key):
    """One pod's worth of the hot path on device ``dev``: stock collect (fused bf16 tcgen05 rollout),
    ppo_update on the SIMT and the tensor-core paths, ppo_update_learners (2 learners, one cluster
    launch), GAE stats, device init, leaderboard stats -- every per-device resource (shared-memory
    attributes, TMA descriptors, image-position tables, scratch) touched."""
    try:
        ctx = pr.Context(dev)
        market = pr.MarketData.synthetic(ctx)
        env = pr.VectorizedEnvironment.stock(ctx, market, pr.StockConfig(), 1500, 2047, 512)
        env.reset(5)
        agent = pr.Agent.init(ctx, 181, 30, seed=7)
        ro = pr.Rollout.for_env(env, 64)
        ro.collect(agent, env, seed=77)
        b = ro.download()
        res = [b["states"], b["actions"], b["log_probs"], b["values"], b["rewards"]]
        cfg = pr.PpoConfig(epochs_per_update=1, minibatch_size=1024, buffer_size=512 * 64)
        for mode in (0, 1):
            agent.set_ppo_mode(mode)
            new, st = pr.ppo_update(agent, ro, cfg, 11)
            res += [new.get()[0], np.array([st.mean_policy_loss, st.mean_value_loss])]
        agent.set_ppo_mode(1)
        outs, stats = pr.ppo_update_learners([agent, agent.clone()], [ro, ro], cfg, [21, 22])
        res += [o.get()[0] for o in outs]
        fresh = pr.Agent(ctx, 181, 30).init_device(99)
        res.append(fresh.get()[0])
        out[key] = res
        ctx.synchronize()
    except BaseException as e:  # surfaced by the caller
        out[key] = e


@pytest.mark.skipif(_gpus() < 2, reason="needs >= 2 GPUs")
def test_two_devices_two_threads_in_process():
    """Multi-device safety in ONE process: the pipeline on device 0 alone, then on devices 0 and 1
    from two threads at once (the C-ABI releases the GIL), each thread's results bit-identical to
    the single-device run -- per-device caches cannot leak a device-0 object into device 1."""
    import threading

    sys.path.insert(0, ROOT)
    from paper_2112_05923_b200 import podracer as pr
    out = {}
    _pipeline(pr, 1, out, "solo1")  # device 1 first: its statics must not be device-0 ones later
    _pipeline(pr, 0, out, "solo0")
    ts = [threading.Thread(target=_pipeline, args=(pr, d, out, f"par{d}")) for d in (0, 1)]
    for t in ts:
        t.start()
    for t in ts:
        t.join(600)
    for k in ("solo0", "solo1", "par0", "par1"):
        assert not isinstance(out[k], BaseException), (k, out[k])
    for k in ("solo1", "par0", "par1"):
        assert len(out[k]) == len(out["solo0"])
        for i, (a, b) in enumerate(zip(out["solo0"], out[k])):
            assert np.array_equal(a, b), (k, i)
