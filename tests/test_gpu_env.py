"""GPU parity: vectorised environments through the C ABI vs the C oracle.

Bar: share counts, dones, resets, episode lengths bit-exact; balances,
rewards and episode returns bit-exact in fp64 before storage (the device
accounting uses the reference's operation order without FMA contraction),
observations/rewards exactly the fp32 rounding of the oracle's fp64 values.
"""
import ctypes as C

import numpy as np
import pytest

from oracle_bind import MT64, StockCfg, ptr, SZ, U8, U64

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pr():
    from paper_2112_05923_b200 import podracer
    return podracer


@pytest.fixture(scope="module")
def ctx(pr):
    return pr.Context(0)


class OracleStockVec:
    def __init__(self, orc, close, ind, cfg, start, end, N):
        self.orc, self.close, self.ind = orc, np.ascontiguousarray(close), np.ascontiguousarray(ind)
        self.K, self.T = close.shape
        self.cfg = StockCfg(cfg.initial_capital, cfg.max_trade_shares, cfg.cost_rate)
        self.start, self.end, self.N = start, end, N
        self.bal = np.zeros(N); self.sh = np.zeros(N * self.K); self.t = np.zeros(N, dtype=np.uint64)
        self.sc = np.zeros(N, dtype=np.uint64); self.er = np.zeros(N)
        orc.orc_stock_vec_reset(N, self.K, C.byref(self.cfg), start, ptr(self.bal), ptr(self.sh), ptr(self.t, SZ),
                                ptr(self.sc, SZ), ptr(self.er))

    def step(self, actions):
        N, K = self.N, self.K
        S = 1 + 6 * K
        nx = np.zeros((N, S)); r = np.zeros(N); d = np.zeros(N, dtype=np.uint8); term = np.zeros((N, S))
        tr = np.zeros(N); tl = np.zeros(N, dtype=np.uint64)
        rc = self.orc.orc_stock_vec_step(N, K, C.byref(self.cfg), self.start, self.end, ptr(self.close),
                                         ptr(self.ind), self.T, ptr(self.bal), ptr(self.sh), ptr(self.t, SZ),
                                         ptr(self.sc, SZ), ptr(self.er),
                                         ptr(np.ascontiguousarray(actions, dtype=np.float64)), ptr(nx), ptr(r),
                                         ptr(d, U8), ptr(term), ptr(tr), ptr(tl, U64))
        assert rc == 0
        return nx, r, d, term, tr, tl


def _market(pr, K, T, seed):
    m = pr.synthetic_market(K, T, seed=seed)
    ind = pr.compute_indicators(m["high"], m["low"], m["close"])
    return m["close"], ind


@pytest.mark.parametrize("K,N,start,end,cfgs", [
    (30, 257, 0, 299, (1e6, 100.0, 0.002)),     # headline shape, ragged last CTA
    (30, 1024, 100, 140, (1e4, 100.0, 0.002)),  # short window: auto-reset every 40 steps, cash-constrained
    (3, 5, 40, 52, (1e3, 1000.0, 0.0)),         # tiny, huge trade sizes, zero cost
    (1, 1, 0, 60, (1000.0, 50.0, 0.002)),
])
def test_stock_vecenv_parity(pr, ctx, orc, K, N, start, end, cfgs):
    T = 300
    close, ind = _market(pr, K, T, seed=11 + K)
    cfg = pr.StockConfig(*cfgs)
    market = pr.MarketData(ctx, close, ind)
    env = pr.VectorizedEnvironment.stock(ctx, market, cfg, start, end, N)
    S = 1 + 6 * K
    assert env.state_dim == S and env.action_dim == K and env.max_episode_steps == end - start
    obs = env.reset(123)
    oracle = OracleStockVec(orc, close, ind, cfg, start, end, N)
    o0 = np.zeros(S)
    orc.orc_stock_observation(cfg.initial_capital, ptr(np.zeros(K)), start, ptr(np.ascontiguousarray(close)),
                              ptr(np.ascontiguousarray(ind)), T, K, C.byref(oracle.cfg), start, ptr(o0))
    assert np.array_equal(obs, np.tile(o0.astype(np.float32), (N, 1)))
    rng = np.random.default_rng(K * 1000 + N)
    n_done = 0
    for step in range(90):
        a = rng.uniform(-1.3, 1.3, size=(N, K)).astype(np.float32)
        if step % 7 == 3:
            a[:, : max(1, K // 3)] = np.nan if step % 14 == 3 else 0.0  # NaN actions trade nothing
        res = env.step(a.astype(np.float64))
        nx, r, d, term, tr, tl = oracle.step(a.astype(np.float64))
        assert np.array_equal(res.dones, d)
        assert np.array_equal(res.next_states, nx.astype(np.float32).astype(np.float64)), f"obs step {step}"
        assert np.array_equal(res.rewards, r.astype(np.float32).astype(np.float64)), f"reward step {step}"
        for i in np.nonzero(d)[0]:
            info = res.infos[i]
            assert info.episode_end and info.episode_length == tl[i]
            assert info.episode_return == tr[i]  # fp64 accumulated on device: bit-exact
            assert np.array_equal(info.terminal_state, term[i].astype(np.float32).astype(np.float64))
        n_done += int(d.sum())
        counts = env.step_counts()
        assert np.all(counts == oracle.sc)
    if end - start < 90:
        assert n_done > 0


def test_stock_vecenv_errors(pr, ctx):
    K, T = 2, 60
    close, ind = _market(pr, K, T, seed=3)
    market = pr.MarketData(ctx, close, ind)
    cfg = pr.StockConfig()
    with pytest.raises(pr.ConfigError):
        pr.VectorizedEnvironment.stock(ctx, market, cfg, 10, 60, 4)  # end >= T (stock_env.hpp:143)
    with pytest.raises(pr.ConfigError):
        pr.VectorizedEnvironment.stock(ctx, market, cfg, 10, 10, 4)
    with pytest.raises(pr.ConfigError):
        pr.VectorizedEnvironment.stock(ctx, market, cfg, 0, 50, 0)  # env.hpp:170
    raw = pr.MarketData(ctx, close, None)
    with pytest.raises(pr.UsageError):
        pr.VectorizedEnvironment.stock(ctx, raw, cfg, 0, 50, 4)  # stock_env.hpp:140
    env = pr.VectorizedEnvironment.stock(ctx, market, cfg, 0, 50, 4)
    with pytest.raises(pr.DimensionError):
        env.step(np.zeros((3, K)))  # env.hpp:201-205
    with pytest.raises(pr.DimensionError):
        env.step(np.zeros((4, K)))  # not reset yet: sub-envs have no state
    env.reset(0)
    env.step(np.zeros((4, K)))


def test_stock_episode_ends_at_window_end(pr, ctx):
    # test_stock_env.cpp:204-218: window [40,45] -> 5 steps
    close, ind = _market(pr, 2, 60, seed=5)
    market = pr.MarketData(ctx, close, ind)
    env = pr.VectorizedEnvironment.stock(ctx, market, pr.StockConfig(), 40, 45, 3)
    env.reset(1)
    steps = 0
    while True:
        res = env.step(np.zeros((3, 2)))
        steps += 1
        if res.dones[0]:
            break
    assert steps == 5 and all(i.episode_length == 5 for i in res.infos)


class OraclePM:
    def __init__(self, orc, N, seed):
        self.orc, self.N = orc, N
        self.g = (MT64 * N)()
        self.st = np.zeros((N, 6)); self.sc = np.zeros(N, dtype=np.uint64); self.er = np.zeros(N)
        orc.orc_pm_vec_reset(N, seed, self.g, ptr(self.st), ptr(self.sc, U64), ptr(self.er))

    def step(self, a):
        N = self.N
        r = np.zeros(N); d = np.zeros(N, dtype=np.uint8); term = np.zeros((N, 6)); tr = np.zeros(N)
        tl = np.zeros(N, dtype=np.uint64)
        self.orc.orc_pm_vec_step(N, self.g, ptr(self.st), ptr(self.sc, U64), ptr(self.er),
                                 ptr(np.ascontiguousarray(a, dtype=np.float64)), ptr(r), ptr(d, U8), ptr(term),
                                 ptr(tr), ptr(tl, U64))
        return r, d, term, tr, tl


@pytest.mark.parametrize("N", [1, 300, 4096])
def test_pointmass_vecenv_parity(pr, ctx, orc, N):
    env = pr.VectorizedEnvironment.pointmass(ctx, N)
    obs = env.reset(77)
    oracle = OraclePM(orc, N, 77)
    # resets drawn from the reference's own per-env mt19937_64 streams (env.hpp:186-194)
    assert np.array_equal(obs, oracle.st.astype(np.float32).astype(np.float64))
    rng = np.random.default_rng(N)
    resets = 0
    for step in range(450):
        a = rng.uniform(-1.5, 1.5, size=(N, 2)).astype(np.float32)
        res = env.step(a.astype(np.float64))
        r, d, term, tr, tl = oracle.step(a.astype(np.float64))
        assert np.array_equal(res.dones, d), f"done step {step}"
        assert np.array_equal(res.rewards, r.astype(np.float32).astype(np.float64))
        assert np.array_equal(res.next_states, oracle.st.astype(np.float32).astype(np.float64)), f"obs step {step}"
        for i in np.nonzero(d)[0]:
            assert res.infos[i].episode_length == tl[i] and res.infos[i].episode_return == tr[i]
            assert np.array_equal(res.infos[i].terminal_state, term[i].astype(np.float32).astype(np.float64))
        resets += int(d.sum())
    assert resets >= N  # every row passed the 200-step limit at least once -> mt streams re-drawn
    assert np.array_equal(env.step_counts(), oracle.sc)


def test_pointmass_reset_deterministic(pr, ctx):
    e1 = pr.VectorizedEnvironment.pointmass(ctx, 8)
    e2 = pr.VectorizedEnvironment.pointmass(ctx, 8)
    s1, s2 = e1.reset(99), e2.reset(99)
    assert np.array_equal(s1, s2)
    assert not np.array_equal(s1, e1.reset(100))  # test_envs.cpp:101-112
    assert np.all(np.abs(s1[:, [0, 1, 4, 5]]) <= 0.4) and np.all(s1[:, [2, 3]] == 0.0)


def test_stock_vecenv_matches_reference_golden(pr, ctx):
    """Device VecEnv against vectors the REFERENCE produced (tests/golden/ref_golden.npz via
    oracle/_ref; env.hpp:167-249, stock_env.hpp:55-184): 30 steps, 6 envs, 12-step episodes
    with auto-reset.  Dones, episode lengths and fp64 episode returns bit-exact; obs and rewards
    are the fp32 rounding of the reference's fp64 values."""
    import os
    g = np.load(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "ref_golden.npz"))
    start, end = (int(x) for x in g["vec_window"])
    close, ind = np.ascontiguousarray(g["vec_close"]), np.ascontiguousarray(g["vec_ind"])
    seq = g["vec_actions"]
    N = seq.shape[1]
    market = pr.MarketData(ctx, close, ind)
    env = pr.VectorizedEnvironment.stock(ctx, market, pr.StockConfig(*(float(x) for x in g["vec_cfg"])), start, end,
                                         N)
    obs = env.reset(9)
    assert np.array_equal(obs, g["vec_obs0"].astype(np.float32))
    f32 = lambda x: x.astype(np.float32).astype(np.float64)
    for s, a in enumerate(seq):
        res = env.step(np.ascontiguousarray(a))
        assert np.array_equal(res.dones, g["vec_done"][s]), f"dones step {s}"
        assert np.array_equal(res.next_states, f32(g["vec_next"][s])), f"obs step {s}"
        assert np.array_equal(res.rewards, f32(g["vec_reward"][s])), f"reward step {s}"
        for i in np.nonzero(g["vec_done"][s])[0]:
            info = res.infos[i]
            assert info.episode_end and info.episode_length == g["vec_term_len"][s][i]
            assert info.episode_return == g["vec_term_ret"][s][i]
            assert np.array_equal(info.terminal_state, f32(g["vec_term"][s][i]))
    assert g["vec_done"].any()


def test_leaderboard_rank_matches_reference_golden(pr, ctx):
    """Device ranking (prb_leaderboard_rank_host) against the final boards the REFERENCE's
    sequential leaderboard_update produced (tournament.hpp:104-119; ties keep the earlier arrival),
    40 sequences of 30 candidates, capacity 1..6: indices bit-exact."""
    import os
    g = np.load(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "ref_golden.npz"))
    for scores, cap, final in zip(g["lb_scores"], g["lb_cap"], g["lb_final"]):
        order = pr.leaderboard_rank(ctx, scores, np.arange(scores.size, dtype=np.uint64), int(cap))
        assert np.array_equal(order.astype(np.int64), final[final >= 0])


def test_leaderboard_stats_matches_reference_golden(pr, ctx):
    """Leaderboard::refresh_stats (tournament.hpp:66-87) on the device: the board the device
    ranking selects from the candidates, then prb_leaderboard_stats over those agents' fp32
    parameter blobs, against the PopulationStats the REFERENCE produced for the same sequence.
    The params are fp32-representable and the device sums in the reference's order in fp64:
    bit-exact."""
    import os
    g = np.load(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "ref_golden_r2.npz"))
    S, A, *hid = (int(x) for x in g["lbs_shape"])
    for c, s, cap, board, m, v in zip(g["lbs_cand"], g["lbs_scores"], g["lbs_cap"], g["lbs_board"], g["lbs_mean"],
                                      g["lbs_var"]):
        order = pr.leaderboard_rank(ctx, s, np.arange(s.size, dtype=np.uint64), int(cap))
        assert np.array_equal(order.astype(np.int64), board[board >= 0])
        agents = []
        for i in order:
            a = pr.Agent(ctx, S, A, hidden=hid)
            a.set(c[i].astype(np.float64))
            agents.append(a)
        st = pr.leaderboard_stats(agents)
        assert np.array_equal(st.mean, m) and np.array_equal(st.variance, v)


def test_leaderboard_stats_stock_board_bit_exact_vs_oracle(pr, ctx, orc):
    """Ten 64x64 stock agents (P = 33,661) on the device: mean / population variance equal the
    oracle's restatement of refresh_stats over the same fp32 parameters bit for bit."""
    from oracle_bind import population_stats
    S, K = 181, 30
    agents = [pr.Agent.init(ctx, S, K, seed=100 + i) for i in range(10)]
    for i, a in enumerate(agents):
        a.mutate(7 + i, 0.05)
    st = pr.leaderboard_stats(agents)
    om, ov = population_stats(orc, [a.flatten_params() for a in agents])
    assert np.array_equal(st.mean, om) and np.array_equal(st.variance, ov)
    assert pr.leaderboard_stats([]).mean.size == 0
