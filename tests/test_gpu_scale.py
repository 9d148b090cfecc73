"""GPU parity at the BASELINE.json shapes (not toy sizes).

Each test runs the product path at a headline configuration and checks a sample of it against
the C oracle (oracle/podracer_oracle.c):

  * configs[1]  stock tcgen05 collect, 30 assets x 65,536 envs x H=256: 512 sampled envs (env 0,
    the last 128-env CTA, random others) replayed on the oracle from their recorded actions --
    states, rewards, dones and final states bit-exact; the bf16 MLP's log-probs and values
    against the oracle's f64 MLP on the same fp32 parameters (stated tolerance below).
  * configs[4]  the same at 1,048,576 envs (a 69 GB buffer): every sampled chunk has rows whose
    float offsets in the time-major buffer exceed 2^32 (steps >= 137).
  * configs[2]  PointMass2D x 262,144 envs x H=256, actor/critic 3x256: 512 sampled envs, resets
    from each env's own mt19937_64 stream (bit-exact), MLP vs the oracle's f64 MLP.
  * GAE (buffer_advantages ppo.hpp:212-244) over the configs[1] buffer: raw advantages / returns
    of the sampled chunks bit-exact fp32 vs the oracle's compute_gae, the whole-buffer mean / std
    within 1e-9 relative of an fp64 host reduction.
  * ppo_update (ppo.hpp:249-296) at 181-64-64-30 / 181-64-64-1, minibatch 1,024, buffer 65,536
    (a real collected buffer), one epoch = 64 Adam steps under the reference's own std::shuffle
    permutation, against orc_ppo_update, plus a teacher-forced 65th step from the device state.

Tolerances for the bf16 tcgen05 rollout MLP, vs the oracle's f64 forward on the same fp32
parameters and observations (bf16 operands with hi+lo pairs for the private obs, fp32
accumulation, tanh.approx):  value |d| <= 5e-2 (1 + |v|),  actor mean |d| <= 5e-2 (1 + |mu|)
(checked through the log-prob: the recorded log-prob is log pi(a | mu_device); the test
recomputes it from the oracle mean with the recorded action and bounds the difference by that
mean tolerance propagated, see _lp_bound). Measured on B200 (stock, configs[1]): value
3.7e-2 (1 + |v|), log-prob 0.26 of the bound; PointMass 3x256 (configs[2]): 1.0e-3, 0.019 -- that
test therefore uses 5e-3.
"""
import ctypes as C

import numpy as np
import pytest

from oracle_bind import MT64, PpoCfg, StockCfg, ptr, SZ, U8, U64

pytestmark = pytest.mark.gpu

K, T_ROWS = 30, 2048
S = 1 + 6 * K


@pytest.fixture(scope="module")
def pr():
    from paper_2112_05923_b200 import podracer
    return podracer


@pytest.fixture(scope="module")
def ctx(pr):
    return pr.Context(0)


def f32(x):
    return np.asarray(x, dtype=np.float32).astype(np.float64)


def dims(*d):
    return np.array(d, dtype=np.uint64)


_CUDART = None


def cudart():
    global _CUDART
    if _CUDART is None:
        for name in ("libcudart.so.12", "libcudart.so", "/usr/local/cuda/lib64/libcudart.so.12"):
            try:
                _CUDART = C.CDLL(name)
                break
            except OSError:
                continue
        _CUDART.cudaMemcpy.argtypes = [C.c_void_p, C.c_void_p, C.c_size_t, C.c_int]
    return _CUDART


def d2h(dptr: int, nbytes: int, dtype) -> np.ndarray:
    out = np.empty(nbytes // np.dtype(dtype).itemsize, dtype=dtype)
    assert cudart().cudaMemcpy(out.ctypes.data, C.c_void_p(dptr), nbytes, 2) == 0  # cudaMemcpyDeviceToHost
    return out


def sample_envs(N, n=512, seed=0):
    rng = np.random.default_rng(seed)
    last_cta = np.arange(max(0, N - 128), N)
    rest = rng.choice(np.arange(1, max(1, N - 128)), size=n - 1 - last_cta.size, replace=False)
    return np.unique(np.concatenate([[0], rest, last_cta])).astype(np.uint64)


def split_flat(S_, A, hidden, flat):
    ad = [S_, *hidden, A]
    pa = sum((i + 1) * o for i, o in zip(ad[:-1], ad[1:]))
    return flat[:pa], flat[pa:pa + A], flat[pa + A:]


def oracle_mlp(orc, params, dims_, X):
    Y = np.zeros((X.shape[0], int(dims_[-1])))
    orc.orc_mlp_forward(ptr(np.ascontiguousarray(params)), ptr(dims_, SZ), len(dims_) - 1,
                        ptr(np.ascontiguousarray(X)), X.shape[0], ptr(Y), None)
    return Y


def _lp_bound(tol_mean, mean, log_std, eps, lp):
    # log pi = sum_d(-0.5 z_d^2 - log_std_d - 0.5 ln 2pi), z_d = (a_d - mu_d)/sigma_d: a mean error
    # delta_d (in sigma units) moves log pi by at most delta_d (|z_d| + delta_d / 2)
    dlt = tol_mean * (1 + np.abs(mean)) / np.exp(log_std)
    return np.sum(dlt * (np.abs(eps) + dlt / 2), axis=1) + 1e-4 * (1 + np.abs(lp))


def check_mlp_vs_oracle(orc, agent, S_, A, hidden, states, actions, log_probs, values, tol, record):
    flat = agent.flatten_params()
    actor, log_std, critic = split_flat(S_, A, hidden, flat)
    mean = oracle_mlp(orc, actor, dims(S_, *hidden, A), states)
    val = oracle_mlp(orc, critic, dims(S_, *hidden, 1), states)[:, 0]
    lp = np.array([orc.orc_gaussian_row_log_prob(ptr(log_std), A, ptr(np.ascontiguousarray(mean[i])),
                                                 ptr(np.ascontiguousarray(actions[i]))) for i in range(len(states))])
    eps = (actions - mean) / np.exp(log_std)
    dv = np.abs(values - val)
    dlp = np.abs(log_probs - lp)
    bound = _lp_bound(tol, mean, log_std, eps, lp)
    record.update(max_dv_rel=float(np.max(dv / (1 + np.abs(val)))), max_dlp=float(np.max(dlp)),
                  max_dlp_over_bound=float(np.max(dlp / bound)))
    import json
    print("RECORD mlp vs oracle f64:", json.dumps(record))
    assert np.all(dv <= tol * (1 + np.abs(val))), record
    assert np.all(dlp <= bound), record


def replay_stock_sample(orc, close, ind, cfg, start, end, n, H, acts):
    c = StockCfg(cfg.initial_capital, cfg.max_trade_shares, cfg.cost_rate)
    bal = np.zeros(n); sh = np.zeros(n * K); t = np.zeros(n, dtype=np.uint64); sc = np.zeros(n, dtype=np.uint64)
    er = np.zeros(n)
    orc.orc_stock_vec_reset(n, K, C.byref(c), start, ptr(bal), ptr(sh), ptr(t, SZ), ptr(sc, SZ), ptr(er))
    states = np.zeros((n, H, S)); rewards = np.zeros((n, H)); dones = np.zeros((n, H), np.uint8)
    obs = np.zeros((n, S))
    for e in range(n):
        orc.orc_stock_observation(bal[e], ptr(np.ascontiguousarray(sh[e * K:(e + 1) * K])), int(t[e]), ptr(close),
                                  ptr(ind), close.shape[1], K, C.byref(c), start, ptr(obs[e]))
    zS, z1, zl = np.zeros((n, S)), np.zeros(n), np.zeros(n, np.uint64)
    for h in range(H):
        states[:, h] = obs
        nx = np.zeros((n, S)); r = np.zeros(n); d = np.zeros(n, np.uint8)
        assert orc.orc_stock_vec_step(n, K, C.byref(c), start, end, ptr(close), ptr(ind), close.shape[1], ptr(bal),
                                      ptr(sh), ptr(t, SZ), ptr(sc, SZ), ptr(er), ptr(np.ascontiguousarray(acts[:, h])),
                                      ptr(nx), ptr(r), ptr(d, U8), ptr(zS), ptr(z1), ptr(zl, U64)) == 0
        rewards[:, h] = r; dones[:, h] = d; obs = nx
    return states, rewards, dones, obs


def stock_market(pr, ctx):
    m = pr.synthetic_market(K, T_ROWS, seed=2112)
    ind = pr.compute_indicators(m["high"], m["low"], m["close"])
    return m, ind, pr.MarketData(ctx, m["close"], ind)


def run_stock_scale(pr, ctx, orc, N, H, start, end, check_mlp, record, check_gae=False):
    m, ind, market = stock_market(pr, ctx)
    cfg = pr.StockConfig()
    env = pr.VectorizedEnvironment.stock(ctx, market, cfg, start, end, N)
    env.reset(2112)
    agent = pr.Agent.init(ctx, S, K, seed=7)
    ro = pr.Rollout.for_env(env, H)
    ro.collect(agent, env, seed=2000)
    envs = sample_envs(N)
    if check_gae:
        ctx.lib.prb_gae(ro.h, 0.99, 0.95, 1)
    b = ro.download_chunks(envs, advantages=check_gae)
    n = envs.size
    acts = b["actions"].reshape(n, H, K)
    st, rw, dn, final = replay_stock_sample(orc, np.ascontiguousarray(m["close"]), np.ascontiguousarray(ind), cfg,
                                            start, end, n, H, acts)
    assert np.array_equal(b["states"], f32(st.reshape(n * H, S))), "states"
    assert np.array_equal(b["rewards"], f32(rw.ravel())), "rewards"
    assert np.array_equal(b["dones"], dn.ravel()), "dones"
    ep = end - start
    if H > ep:
        assert dn[:, ep - 1].all()
    # final VecEnv states of the sampled envs (states() rows on the device)
    dobs = env.states_device_ptr()
    fin = np.stack([d2h(dobs + int(e) * S * 4, S * 4, np.float32) for e in envs]).astype(np.float64)
    assert np.array_equal(fin, f32(final)), "final states"
    # the sampled chunks include transitions whose float offsets in the time-major buffer exceed 2^32
    record["max_obs_float_offset"] = int(((H - 1) * N + int(envs[-1])) * (1 + K))
    record["max_act_float_offset"] = int(((H - 1) * N + int(envs[-1])) * K)
    if check_mlp:
        check_mlp_vs_oracle(orc, agent, S, K, (64, 64), b["states"], b["actions"], b["log_probs"], b["values"], 5e-2,
                            record)
        # bootstrap V(s_H) of the sampled envs vs the oracle critic on the final states
        _, _, critic = split_flat(S, K, (64, 64), agent.flatten_params())
        vb = oracle_mlp(orc, critic, dims(S, 64, 64, 1), f32(final))[:, 0]
        assert np.all(np.abs(b["bootstrap"] - vb) <= 5e-2 * (1 + np.abs(vb)))
    if check_gae:
        adv = np.zeros(n * H); ret = np.zeros(n * H)
        for i in range(n):
            sl = slice(i * H, (i + 1) * H)
            orc.orc_compute_gae(ptr(np.ascontiguousarray(b["rewards"][sl])), ptr(np.ascontiguousarray(b["values"][sl])),
                                ptr(np.ascontiguousarray(b["dones"][sl]), U8), H, float(b["bootstrap"][i]), 0.99, 0.95,
                                ptr(adv[sl]), ptr(ret[sl]))
        assert np.array_equal(b["raw_advantages"], f32(adv)), "raw advantages"
        assert np.array_equal(b["returns"], f32(ret)), "returns"
        # whole-buffer normalisation (ppo.hpp:234-242) vs an fp64 host reduction of the device's
        # own raw advantages (fp32 values, time-major [H][N] array)
        fields = [C.c_void_p() for _ in range(7)]
        ctx.lib.prb_rollout_device_fields(ro.h, *[C.byref(f) for f in fields])
        mean, denom = ro.gae_stats()
        # the statistics cover every transition: recompute all raw advantages from the full
        # reward / value / done arrays with the oracle, one chunk at a time
        rew = d2h(fields[3].value, N * H * 4, np.float32).reshape(H, N).T.astype(np.float64)
        val = d2h(fields[4].value, N * H * 4, np.float32).reshape(H, N).T.astype(np.float64)
        don = d2h(fields[5].value, N * H, np.uint8).reshape(H, N).T.copy()
        boot = d2h(fields[6].value, N * 4, np.float32).astype(np.float64)
        full = np.zeros((N, H)); fr = np.zeros(H)
        for e in range(N):
            orc.orc_compute_gae(ptr(np.ascontiguousarray(rew[e])), ptr(np.ascontiguousarray(val[e])),
                                ptr(np.ascontiguousarray(don[e]), U8), H, float(boot[e]), 0.99, 0.95, ptr(full[e]),
                                ptr(fr))
        a32 = f32(full)
        mu = a32.mean()
        sd = max(np.sqrt(np.mean((a32 - mu) ** 2)), 1e-8)
        record.update(gae_mean=mean, gae_denom=denom, host_mean=float(mu), host_sd=float(sd))
        assert abs(mean - mu) <= 1e-9 * max(1.0, abs(mu)) + 1e-12 * sd, record
        assert abs(denom - sd) <= 1e-9 * sd, record
    del ro
    return record


def test_stock_collect_configs1_sampled_replay(pr, ctx, orc):
    """configs[1]: 65,536 envs x 256 with episodes of 147 steps (resets inside the horizon),
    512 sampled envs bit-exact on the oracle, bf16 MLP vs oracle f64, GAE of the same buffer."""
    rec = run_stock_scale(pr, ctx, orc, 65536, 256, 1900, 2047, True, {}, check_gae=True)
    print("RECORD configs[1]", rec)


def test_stock_collect_configs4_sampled_replay_beyond_2_32(pr, ctx, orc):
    """configs[4]: 1,048,576 envs x 256 (69 GB rollout buffer): the sampled chunks' rows beyond
    step 137 sit past 2^32 floats into the obs / action arrays; transitions bit-exact."""
    rec = run_stock_scale(pr, ctx, orc, 1 << 20, 256, 0, 2047, False, {})
    assert rec["max_obs_float_offset"] > (1 << 32) and rec["max_act_float_offset"] > (1 << 32)
    print("RECORD configs[4]", rec)


def test_pointmass_collect_configs2_sampled_replay(pr, ctx, orc):
    """configs[2]: PointMass2D x 262,144 envs x 256, 3x256 actor/critic on tcgen05; 512 sampled
    envs replayed on the oracle with their own reset streams (derive_seed(seed, kVecEnv, e)),
    bit-exact states / rewards / dones / step counts; MLP vs the oracle's f64 forward."""
    N, H = 262144, 256
    env = pr.VectorizedEnvironment.pointmass(ctx, N)
    env.reset(3)
    agent = pr.Agent.init(ctx, 6, 2, seed=4, hidden=(256, 256, 256))
    ro = pr.Rollout.for_env(env, H)
    ro.collect(agent, env, seed=8)
    envs = sample_envs(N, seed=1)
    n = envs.size
    b = ro.download_chunks(envs)
    gens = (MT64 * n)()
    st = np.zeros((n, 6)); sc = np.zeros(n, np.uint64); er = np.zeros(n)
    orc.orc_pm_vec_reset_subset(n, ptr(envs, U64), 3, gens, ptr(st), ptr(sc, U64), ptr(er))
    states = b["states"].reshape(n, H, 6); acts = b["actions"].reshape(n, H, 2)
    rw, dn = b["rewards"].reshape(n, H), b["dones"].reshape(n, H)
    z6, z1, zl = np.zeros((n, 6)), np.zeros(n), np.zeros(n, np.uint64)
    for h in range(H):
        assert np.array_equal(states[:, h], f32(st)), h
        r = np.zeros(n); d = np.zeros(n, np.uint8)
        orc.orc_pm_vec_step(n, gens, ptr(st), ptr(sc, U64), ptr(er), ptr(np.ascontiguousarray(acts[:, h])), ptr(r),
                            ptr(d, U8), ptr(z6), ptr(z1), ptr(zl, U64))
        assert np.array_equal(rw[:, h], f32(r)), h
        assert np.array_equal(dn[:, h], d), h
    assert dn.sum() >= n  # 200-step limit inside the horizon
    dobs = env.states_device_ptr()
    fin = np.stack([d2h(dobs + int(e) * 6 * 4, 24, np.float32) for e in envs]).astype(np.float64)
    assert np.array_equal(fin, f32(st))
    rec = {}
    check_mlp_vs_oracle(orc, agent, 6, 2, (256, 256, 256), b["states"], b["actions"], b["log_probs"], b["values"],
                        5e-3, rec)
    print("RECORD configs[2]", rec)
    del ro


def orc_update(orc, p, m, v, t, buf, rows, N, H, epochs, mb, perms):
    """orc_ppo_update (f64) in place on (p, m, v); returns (t, [policy, value, entropy, steps])."""
    tt = C.c_int64(t); so = np.zeros(4)
    sl = {k: np.ascontiguousarray(buf[k][rows]) for k in ("states", "actions", "log_probs", "rewards", "dones",
                                                         "values")}
    offs = np.arange(N, dtype=np.uint64) * H; lens = np.full(N, H, dtype=np.uint64)
    oc = PpoCfg(0.99, 0.95, 0.2, 0.01, 0.5, epochs, mb, N * H, 1e-3)
    assert orc.orc_ppo_update(ptr(p), ptr(m), ptr(v), C.byref(tt), ptr(dims(S, 64, 64, K), SZ), 3,
                              ptr(dims(S, 64, 64, 1), SZ), 3, ptr(sl["states"]), ptr(sl["actions"]),
                              ptr(sl["log_probs"]), ptr(sl["rewards"]), ptr(sl["dones"], U8), ptr(sl["values"]),
                              N * H, S, ptr(offs, SZ), ptr(lens, SZ), ptr(np.ascontiguousarray(buf["bootstrap"][:N])),
                              N, C.byref(oc), ptr(perms, U64), ptr(so)) == 0
    return tt.value, so


def test_ppo_update_headline_shape_vs_oracle(pr, ctx, orc, ref):
    """ppo_update at the headline net (181-64-64-30 / 181-64-64-1), minibatch 1,024, on a real
    collected buffer of 65,536 transitions (256 envs x 256 steps, old log-probs = the oracle's f64
    values, so the first ratio is exactly 1 as in the reference), one epoch = 64 sequential Adam
    steps under the reference's own std::shuffle permutation, against orc_ppo_update (f64), for
    both device paths (fp32 SIMT, mode 0; tensor cores, mode 1).

    Part 1, 64 free-running steps. The stock observation is unnormalised (prices and holdings in
    the thousands), so a W1 change of lr moves a pre-activation by O(1): within a few steps the
    ratios leave [0.8, 1.2], the actor's gradient comes from whichever samples sit inside the clip
    range, and the actor's trajectory is chaotic under rounding -- measured for the fp32 SIMT path,
    the device and f64 actor updates end uncorrelated (|dp| ~ |update|) while the critic, whose
    loss is smooth, stays within 3% and its Adam moments within 0.3%. Bounded: the critic's
    parameters and moments, the mean value loss and entropy, the policy loss within 10%, the
    actor's update norm within 25% of the oracle's.
    Part 2, teacher-forced step 65 at the drifted state (ratios far from 1, the clip active): from
    the device state after part 1, one more minibatch (envs 0-3, 1,024 transitions) on the device
    and on the oracle from the SAME (params, m, v, t); the update vectors must agree to a small
    fraction (measured: SIMT 7.4e-6, tensor cores 3.9e-3 relative) -- the per-step precision claim at the headline shape."""
    N, H = 256, 256
    n = N * H
    m, ind, market = stock_market(pr, ctx)
    env = pr.VectorizedEnvironment.stock(ctx, market, pr.StockConfig(), 1500, 2047, N)
    env.reset(5)
    agent = pr.Agent.init(ctx, S, K, seed=7)
    ro0 = pr.Rollout.for_env(env, H)
    ro0.collect(agent, env, seed=77)
    buf = ro0.download()
    flat = agent.flatten_params()
    actor, log_std, _ = split_flat(S, K, (64, 64), flat)
    pa = actor.size + K  # actor + log_std | critic
    mean = oracle_mlp(orc, actor, dims(S, 64, 64, K), buf["states"])
    buf["log_probs"] = np.array([orc.orc_gaussian_row_log_prob(ptr(log_std), K, ptr(np.ascontiguousarray(mean[i])),
                                                               ptr(np.ascontiguousarray(buf["actions"][i])))
                                 for i in range(n)])
    ro = pr.Rollout.raw(ctx, N, H, S, K)
    ro.upload(buf["states"], buf["actions"], buf["log_probs"], buf["rewards"], buf["dones"], buf["values"],
              buf["bootstrap"])
    N1 = 4  # part 2 sub-buffer: envs 0..3 (rows are env-major in the download)
    ro1 = pr.Rollout.raw(ctx, N1, H, S, K)
    r1 = slice(0, N1 * H)
    ro1.upload(*(np.ascontiguousarray(buf[k][r1]) for k in ("states", "actions", "log_probs", "rewards", "dones",
                                                            "values")), np.ascontiguousarray(buf["bootstrap"][:N1]))
    epochs, mb, seed = 1, 1024, 4242
    perms = np.zeros(epochs * n, dtype=np.uint64)
    ref.ref_ppo_permutations(seed, n, epochs, ptr(perms, U64))
    perm1 = np.zeros(mb, dtype=np.uint64)
    ref.ref_ppo_permutations(seed + 1, mb, 1, ptr(perm1, U64))
    cfg = pr.PpoConfig(epochs_per_update=epochs, minibatch_size=mb, buffer_size=n)
    cfg1 = pr.PpoConfig(epochs_per_update=1, minibatch_size=mb, buffer_size=mb)
    fo, mo, vo = flat.copy(), np.zeros(flat.size), np.zeros(flat.size)
    to, so = orc_update(orc, fo, mo, vo, 0, buf, slice(0, n), N, H, epochs, mb, perms)
    steps = epochs * (n // mb)
    rl2 = lambda x, y: float(np.linalg.norm(x - y) / np.linalg.norm(y))
    for mode, tol_critic, tol65 in ((0, 0.05, 1e-4), (1, 0.1, 0.02)):  # measured 0.029/7.4e-6, 0.050/3.9e-3
        agent.set_ppo_mode(mode)
        new, stats = pr.ppo_update(agent, ro, cfg, seed, perm=perms)
        p, mm, vv, t = new.get()
        r = dict(actor_rel=float(np.linalg.norm((p - fo)[:pa]) / np.linalg.norm((fo - flat)[:pa])),
                 critic_rel=float(np.linalg.norm((p - fo)[pa:]) / np.linalg.norm((fo - flat)[pa:])),
                 m_actor=rl2(mm[:pa], mo[:pa]), m_critic=rl2(mm[pa:], mo[pa:]),
                 v_actor=rl2(vv[:pa], vo[:pa]), v_critic=rl2(vv[pa:], vo[pa:]),
                 pl=(stats.mean_policy_loss, so[0]), vl=(stats.mean_value_loss, so[1]),
                 ent=(stats.mean_entropy, so[2]))
        assert t == to == steps and stats.minibatches == so[3] == steps
        # part 2: one teacher-forced step from the device state
        a2 = pr.Agent(ctx, S, K)
        a2.set(p, mm, vv, t)
        a2.set_ppo_mode(mode)
        n2, st2 = pr.ppo_update(a2, ro1, cfg1, seed + 1, perm=perm1)
        p2, m2, v2, t2 = n2.get()
        fo2, mo2, vo2 = p.copy(), mm.copy(), vv.copy()
        t2o, so2 = orc_update(orc, fo2, mo2, vo2, t, buf, r1, N1, H, 1, mb, perm1)
        dd, do = p2 - p, fo2 - p
        r["step65_max_over_lr"] = float(np.max(np.abs(dd - do)) / 1e-3)
        r["step65_rel"] = rl2(dd, do)
        r["step65_pl"] = (st2.mean_policy_loss, so2[0])
        assert t2 == t2o == t + 1
        r["actor_update_norm_ratio"] = float(np.linalg.norm((p - flat)[:pa]) / np.linalg.norm((fo - flat)[:pa]))
        print(f"RECORD ppo_update headline mode {mode}: {r}")
        assert r["m_critic"] <= 0.01 and r["v_critic"] <= 0.01 and r["critic_rel"] <= tol_critic
        un = r["actor_update_norm_ratio"]
        assert 0.8 <= un <= 1.25 and np.isfinite(p).all()
        assert abs(stats.mean_policy_loss - so[0]) <= 0.1 * abs(so[0])
        assert abs(stats.mean_value_loss - so[1]) <= 1e-5 * abs(so[1])
        assert abs(stats.mean_entropy - so[2]) <= 1e-3 * abs(so[2])
        assert r["step65_rel"] <= tol65
        assert abs(st2.mean_policy_loss - so2[0]) <= 1e-3 * (1 + abs(so2[0]))
    agent.set_ppo_mode(0)
    assert np.array_equal(agent.flatten_params(), flat)  # purity (ppo.hpp:246-248)
