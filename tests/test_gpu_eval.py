"""GPU: the device evaluator (evaluate pod.hpp:43-83) against the oracle.

The evaluator resets one env per episode with derive_seed(seed, kEpisode, i)
and plays the policy mean clipped to the spec bounds.  The oracle side replays
the same suite with the oracle's env transitions (bit-exact with the
reference) driven by the device's own fp32 policy mean on the oracle's states
(the evaluator's policy input), so every episode total and length must match
EXACTLY; mean / population std follow EvaluationRecord (pod.hpp:76-81)."""
import ctypes as C

import numpy as np
import pytest

from oracle_bind import MT64, StockCfg, ptr, D, SZ, U8, U64, derive_seed

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pr():
    from paper_2112_05923_b200 import podracer
    return podracer


@pytest.fixture(scope="module")
def ctx(pr):
    return pr.Context(0)


def _stats(r):
    m = sum(r) / len(r)
    return m, (sum((x - m) * (x - m) for x in r) / len(r)) ** 0.5


@pytest.mark.parametrize("hidden", [(64, 64), (256, 256, 256)])
def test_evaluate_pointmass_matches_oracle(pr, ctx, orc, hidden):
    E, seed = 10, 2112
    agent = pr.Agent.init(ctx, 6, 2, seed=5, hidden=hidden)
    env = pr.VectorizedEnvironment.pointmass(ctx, E)
    rec = pr.evaluate(agent, env, seed)
    gens = (MT64 * E)()
    st = np.zeros((E, 6)); sc = np.zeros(E, np.uint64); er = np.zeros(E)
    for e in range(E):
        orc.orc_mt64_seed(C.byref(gens[e]), derive_seed(orc, seed, 8, e))  # kEpisode stream (pod.hpp:52)
        orc.orc_pointmass_reset(C.byref(gens[e]), ptr(st[e]))
    first_ret, first_len = [None] * E, [0] * E
    for _ in range(200):
        mean = agent.policy_mean(st.astype(np.float32))
        acts = np.clip(mean.astype(np.float64), -1.0, 1.0)
        r = np.zeros(E); d = np.zeros(E, np.uint8); tr = np.zeros(E); tl = np.zeros(E, np.uint64)
        orc.orc_pm_vec_step(E, gens, ptr(st), ptr(sc, U64), ptr(er), ptr(np.ascontiguousarray(acts)), ptr(r),
                            ptr(d, U8), ptr(np.zeros((E, 6))), ptr(tr), ptr(tl, U64))
        for e in range(E):
            if d[e] and first_ret[e] is None:
                first_ret[e], first_len[e] = tr[e], int(tl[e])
    assert all(x is not None for x in first_ret)
    assert np.array_equal(rec.episodic_rewards, np.array(first_ret))
    assert rec.eval_steps == sum(first_len)
    m, sd = _stats(first_ret)
    assert rec.mean == pytest.approx(m, rel=1e-15, abs=1e-12) and rec.std_dev == pytest.approx(sd, rel=1e-12, abs=1e-12)
    # a fixed seed defines a fixed suite; a different seed a different one
    assert np.array_equal(pr.evaluate(agent, env, seed).episodic_rewards, rec.episodic_rewards)
    assert not np.array_equal(pr.evaluate(agent, env, seed + 1).episodic_rewards, rec.episodic_rewards)


def test_evaluate_stock_matches_oracle(pr, ctx, orc):
    K, T, E, seed = 30, 120, 3, 7
    m = pr.synthetic_market(K, T, seed=2112)
    ind = pr.compute_indicators(m["high"], m["low"], m["close"])
    market = pr.MarketData(ctx, m["close"], ind)
    cfg = pr.StockConfig()
    start, end = 10, 50
    S = 1 + 6 * K
    agent = pr.Agent.init(ctx, S, K, seed=3)
    env = pr.VectorizedEnvironment.stock(ctx, market, cfg, start, end, E)
    rec = pr.evaluate(agent, env, seed)
    close, indc = np.ascontiguousarray(m["close"]), np.ascontiguousarray(ind)
    c = StockCfg(cfg.initial_capital, cfg.max_trade_shares, cfg.cost_rate)
    bal = np.zeros(E); sh = np.zeros(E * K); t = np.zeros(E, dtype=np.uint64); sc = np.zeros(E, dtype=np.uint64)
    er = np.zeros(E)
    orc.orc_stock_vec_reset(E, K, C.byref(c), start, ptr(bal), ptr(sh), ptr(t, SZ), ptr(sc, SZ), ptr(er))
    obs = np.zeros((E, S))
    for e in range(E):
        orc.orc_stock_observation(bal[e], ptr(np.ascontiguousarray(sh[e * K:(e + 1) * K])), int(t[e]), ptr(close),
                                  ptr(indc), T, K, C.byref(c), start, ptr(obs[e]))
    first_ret, first_len = [None] * E, [0] * E
    for _ in range(end - start):
        acts = np.clip(agent.policy_mean(obs.astype(np.float32)).astype(np.float64), -1.0, 1.0)
        nx = np.zeros((E, S)); r = np.zeros(E); d = np.zeros(E, np.uint8); tr = np.zeros(E)
        tl = np.zeros(E, np.uint64)
        orc.orc_stock_vec_step(E, K, C.byref(c), start, end, ptr(close), ptr(indc), T, ptr(bal), ptr(sh),
                               ptr(t, SZ), ptr(sc, SZ), ptr(er), ptr(np.ascontiguousarray(acts)), ptr(nx), ptr(r),
                               ptr(d, U8), ptr(np.zeros((E, S))), ptr(tr), ptr(tl, U64))
        for e in range(E):
            if d[e] and first_ret[e] is None:
                first_ret[e], first_len[e] = tr[e], int(tl[e])
        obs = nx
    assert np.array_equal(rec.episodic_rewards, np.array(first_ret))
    assert rec.eval_steps == sum(first_len) == E * (end - start)
    assert rec.std_dev == 0.0  # the stock reset ignores the stream: identical episodes


def test_evaluate_errors(pr, ctx):
    agent = pr.Agent.init(ctx, 6, 2, seed=5)
    wrong = pr.Agent.init(ctx, 5, 2, seed=5)
    env = pr.VectorizedEnvironment.pointmass(ctx, 4)
    with pytest.raises(pr.DimensionError):
        pr.evaluate(wrong, env, 1)
    rec = pr.evaluate(agent, env, 1, sample_actions=True)  # Philox-sampled actions: statistics only
    assert np.all(np.isfinite(rec.episodic_rewards)) and 4 <= rec.eval_steps <= 800


@pytest.mark.parametrize("kind,sample", [("stock", False), ("pointmass", True), ("pointmass", False)])
def test_evaluate_pods_equals_per_pod_evaluate(pr, ctx, kind, sample):
    """prb_evaluate_pods (one policy launch per step for every pod) gives each pod exactly the
    record prb_evaluate gives it alone: episode totals, lengths, mean, std."""
    P, E = 3, 10
    if kind == "stock":
        market = pr.MarketData.synthetic(ctx)
        mk = lambda: pr.VectorizedEnvironment.stock(ctx, market, pr.StockConfig(), 1900, 1940, E)  # noqa: E731
        agents = [pr.Agent.init(ctx, 181, 30, seed=20 + p) for p in range(P)]
    else:
        mk = lambda: pr.VectorizedEnvironment.pointmass(ctx, E)  # noqa: E731
        agents = [pr.Agent.init(ctx, 6, 2, seed=20 + p) for p in range(P)]
    seeds = [100 + 7 * p for p in range(P)]
    grouped = pr.evaluate_pods(agents, [mk() for _ in range(P)], seeds, sample_actions=sample)
    for p in range(P):
        one = pr.evaluate(agents[p], mk(), seeds[p], sample_actions=sample)
        assert np.array_equal(grouped[p].episodic_rewards, one.episodic_rewards), p
        assert grouped[p].mean == one.mean and grouped[p].std_dev == one.std_dev
        assert grouped[p].eval_steps == one.eval_steps


def test_evaluate_pods_errors(pr, ctx):
    """prb_evaluate_pods rejects pods whose eval VecEnvs differ in shape (UsageError) and agents that
    do not match their envs (DimensionError); P = 0 is a no-op."""
    a = pr.Agent.init(ctx, 6, 2, seed=1)
    e10, e12 = pr.VectorizedEnvironment.pointmass(ctx, 10), pr.VectorizedEnvironment.pointmass(ctx, 12)
    with pytest.raises(pr.UsageError):
        pr.evaluate_pods([a, a], [e10, e12], [1, 2])
    market = pr.MarketData.synthetic(ctx)
    stock = pr.VectorizedEnvironment.stock(ctx, market, pr.StockConfig(), 1900, 1940, 10)
    with pytest.raises((pr.DimensionError, pr.UsageError)):
        pr.evaluate_pods([a], [stock], [1])
    assert pr.evaluate_pods([], [], []) == []
