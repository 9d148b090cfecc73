"""GPU: the pod population of BASELINE configs[3] on one device.

  * prb_rollout_collect_pods (every pod's collect in ONE tcgen05 launch, per-pod weights) gives
    bit-identical buffers and VecEnv states to one prb_rollout_collect per pod.
  * PodPopulation.generation (tournament.py: grouped collect -> concurrent learners on the tensor
    cores -> per-pod fusion -> evaluation -> device ranking -> elite copies + mutation) runs,
    its board is the reference ordering of the scores (tournament.hpp:104-119), and it is
    deterministic for a fixed seed.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu
K, S = 30, 181


@pytest.fixture(scope="module")
def pr():
    from paper_2112_05923_b200 import podracer
    return podracer


@pytest.fixture(scope="module")
def ctx(pr):
    return pr.Context(0)


@pytest.fixture(scope="module")
def market(pr, ctx):
    m = pr.synthetic_market(K, 512, seed=2112)
    ind = pr.compute_indicators(m["high"], m["low"], m["close"])
    return pr.MarketData(ctx, m["close"], ind)


def test_grouped_collect_equals_per_pod_collects(pr, ctx, market):
    P, N, H = 3, 300, 40  # N not a multiple of the 128-env tile; episodes end inside the horizon
    envs_a = [pr.VectorizedEnvironment.stock(ctx, market, pr.StockConfig(), 100, 130, N) for _ in range(P)]
    envs_b = [pr.VectorizedEnvironment.stock(ctx, market, pr.StockConfig(), 100, 130, N) for _ in range(P)]
    agents = [pr.Agent.init(ctx, S, K, seed=10 + p) for p in range(P)]
    seeds = [77 + p for p in range(P)]
    for p in range(P):
        envs_a[p].reset(p)
        envs_b[p].reset(p)
    ro_a = [pr.Rollout.for_env(e, H) for e in envs_a]
    ro_b = [pr.Rollout.for_env(e, H) for e in envs_b]
    for _ in range(2):  # twice: the second collect starts from the first one's final states
        pr.collect_pods(ro_a, agents, envs_a, seeds)
        for p in range(P):
            ro_b[p].set_mode(2)
            ro_b[p].collect(agents[p], envs_b[p], seeds[p])
        for p in range(P):
            a, b = ro_a[p].download(), ro_b[p].download()
            for key in a:
                assert np.array_equal(a[key], b[key]), (p, key)
            assert np.array_equal(envs_a[p].states(), envs_b[p].states())
    assert not np.array_equal(ro_a[0].download()["actions"], ro_a[1].download()["actions"])


def test_pod_population_generation(pr, ctx, market):
    from paper_2112_05923_b200 import tournament as tn
    P, N, H, L = 4, 128, 32, 2
    cfg = pr.PpoConfig(minibatch_size=1024, epochs_per_update=1, buffer_size=N * H)

    def run():
        pop = tn.PodPopulation(ctx, market, pr.StockConfig(), pods=P, envs_per_pod=N, horizon=H, learners=L,
                               ppo_cfg=cfg, window=(0, 400), eval_episodes=4, eval_window=(300, 340), capacity=3,
                               top_k=2, seed=5)
        return [pop.generation() for _ in range(2)], pop
    out1, pop = run()
    out2, _ = run()
    assert out1 == out2  # deterministic
    for g in out1:
        s = np.array(g["scores"])
        assert np.all(np.isfinite(s)) and g["minibatches_per_learner"] == (N * H) // 1024
        seqs = [tn.arrival_seq(g["generation"], p, P) for p in range(P)]
        assert g["board"] == tn.rank_candidates_host(s, seqs, 3)
    assert all(np.all(np.isfinite(a.flatten_params())) for a in pop.agents)


def test_collect_pods_other_envs_fall_back(pr, ctx):
    """prb_rollout_collect_pods with pods the grouped stock kernel does not take (PointMass): each
    pod is collected on its own path, identical to prb_rollout_collect."""
    agents = [pr.Agent.init(ctx, 6, 2, seed=30 + p, hidden=(64, 64)) for p in range(2)]
    envs_a = [pr.VectorizedEnvironment.pointmass(ctx, 64) for _ in range(2)]
    envs_b = [pr.VectorizedEnvironment.pointmass(ctx, 64) for _ in range(2)]
    for p in range(2):
        envs_a[p].reset(40 + p)
        envs_b[p].reset(40 + p)
    ro_a = [pr.Rollout.for_env(e, 16) for e in envs_a]
    ro_b = [pr.Rollout.for_env(e, 16) for e in envs_b]
    pr.collect_pods(ro_a, agents, envs_a, [50, 51])
    for p in range(2):
        ro_b[p].collect(agents[p], envs_b[p], seed=50 + p)
        da, db = ro_a[p].download(), ro_b[p].download()
        assert all(np.array_equal(da[k], db[k]) for k in ("states", "actions", "rewards", "dones"))
