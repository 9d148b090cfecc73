"""GPU parity of the tensor-core PPO update (ppo_tc.cu: one thread-block cluster per learner) and
the concurrent-learner entry point prb_ppo_update_learners (pod.hpp:436-461).

Precision: bf16 MMA operands (inputs AND first-layer weights as hi + lo bf16 pairs in the forward),
fp32 accumulation and
fp32 elementwise head / Adam math.  Stated tolerances, vs the C oracle's f64 detail::ppo_loss_grads
on the same fp32 parameters and rows (ppo.hpp:116-188), per parameter block b of the flat layout:
    relative L2 error  |g_b - g_orc_b| / |g_orc_b|  <=  2e-2   (measured max 0.76%, actor layer 1)
with the old log-probs set to the oracle's own f64 log-probs, so a ratio differs from 1 only by the
device forward's rounding (the reference's first minibatch has ratio == 1 exactly).
"""
import ctypes as C

import numpy as np
import pytest

from oracle_bind import PpoCfg, ptr, SZ, U8, U64

pytestmark = pytest.mark.gpu

K, S = 30, 181
TOL_BLOCK = 2e-2


@pytest.fixture(scope="module")
def pr():
    from paper_2112_05923_b200 import podracer
    return podracer


@pytest.fixture(scope="module")
def ctx(pr):
    return pr.Context(0)


def dims(*d):
    return np.array(d, dtype=np.uint64)


def blocks(A, hidden=(64, 64)):
    out, off = [], 0
    for net, n_out in (("a", A), ("c", 1)):
        d = [S, *hidden, n_out]
        for l in range(3):
            i, o = d[l], d[l + 1]
            out += [(f"{net}.W{l + 1}", off, off + i * o), (f"{net}.b{l + 1}", off + i * o, off + i * o + o)]
            off += i * o + o
        if net == "a":
            out.append(("log_std", off, off + A))
            off += A
    return out


def oracle_logp(orc, flat, states, actions):
    pa = sum((i + 1) * o for i, o in zip([S, 64, 64], [64, 64, K]))
    actor, ls = flat[:pa], flat[pa:pa + K]
    mean = np.zeros((len(states), K))
    orc.orc_mlp_forward(ptr(np.ascontiguousarray(actor)), ptr(dims(S, 64, 64, K), SZ), 3,
                        ptr(np.ascontiguousarray(states)), len(states), ptr(mean), None)
    return np.array([orc.orc_gaussian_row_log_prob(ptr(ls), K, ptr(np.ascontiguousarray(mean[i])),
                                                   ptr(np.ascontiguousarray(actions[i]))) for i in range(len(states))])


def real_buffer(pr, ctx, orc, N, H, agent, seed=77, oracle_lp=True):
    """A collected stock buffer uploaded as full rows, old log-probs = the oracle's f64 log-probs."""
    m = pr.synthetic_market(K, 2048, 2112)
    ind = pr.compute_indicators(m["high"], m["low"], m["close"])
    market = pr.MarketData(ctx, m["close"], ind)
    env = pr.VectorizedEnvironment.stock(ctx, market, pr.StockConfig(), 1500, 2047, N)
    env.reset(5)
    ro = pr.Rollout.for_env(env, H)
    ro.collect(agent, env, seed=seed)
    b = ro.download()
    if oracle_lp:
        b["log_probs"] = oracle_logp(orc, agent.flatten_params(), b["states"], b["actions"])
    raw = pr.Rollout.raw(ctx, N, H, S, K)
    raw.upload(b["states"], b["actions"], b["log_probs"], b["rewards"], b["dones"], b["values"], b["bootstrap"])
    return raw, b


def test_tc_gradient_blocks_vs_oracle(pr, ctx, orc):
    """One minibatch step of 1,024 rows (8 CTAs), lr = 0: the reduced gradient of every parameter
    block against orc_ppo_loss_grads on the same rows within TOL_BLOCK relative L2."""
    N, H, mb = 16, 64, 1024
    n = N * H
    agent = pr.Agent.init(ctx, S, K, seed=7)
    agent.set_ppo_mode(1)
    ro, b = real_buffer(pr, ctx, orc, N, H, agent)
    perm = np.random.default_rng(3).permutation(n).astype(np.uint64)
    cfg = pr.PpoConfig(epochs_per_update=1, minibatch_size=mb, buffer_size=n, learning_rate=0.0)
    out = pr.Agent(ctx, S, K)
    pr.ppo_update(agent, ro, cfg, 1, perm=perm, out=out)
    g = np.zeros(agent.param_count)
    ctx.lib.prb_debug_agent_grads(out.h, g.ctypes.data_as(C.POINTER(C.c_double)))
    adv, ret = ro.buffer_advantages(cfg, normalize=True)
    idx = perm[:mb].astype(np.int64)
    flat = agent.flatten_params()
    og, ol = np.zeros(flat.size), np.zeros(3)
    oc = PpoCfg(0.99, 0.95, 0.2, 0.01, 0.5, 1, mb, n, 0.0)
    assert orc.orc_ppo_loss_grads(ptr(flat), ptr(dims(S, 64, 64, K), SZ), 3, ptr(dims(S, 64, 64, 1), SZ), 3,
                                  ptr(np.ascontiguousarray(b["states"][idx])),
                                  ptr(np.ascontiguousarray(b["actions"][idx])),
                                  ptr(np.ascontiguousarray(b["log_probs"][idx])), ptr(np.ascontiguousarray(adv[idx])),
                                  ptr(np.ascontiguousarray(ret[idx])), mb, C.byref(oc), ptr(og), ptr(ol)) == 0
    errs = {}
    for name, lo, hi in blocks(K):
        ref = og[lo:hi]
        errs[name] = float(np.linalg.norm(g[lo:hi] - ref) / max(np.linalg.norm(ref), 1e-30))
    print("RECORD tc gradient rel L2 per block:", errs)
    assert max(errs.values()) <= TOL_BLOCK, errs


def test_tc_update_vs_oracle_and_simt(pr, ctx, orc, ref):
    """A 4-step update (buffer 4,096, minibatch 1,024) under the reference's own std::shuffle
    permutation: the tensor-core result against orc_ppo_update, and the SIMT path's result against
    the same oracle -- the tensor-core update's distance from the oracle is within 3x the fp32
    SIMT update's plus the bf16 allowance, and the mean losses agree to 1e-2 relative."""
    N, H, mb, epochs = 16, 256, 1024, 1
    n = N * H
    agent = pr.Agent.init(ctx, S, K, seed=7)
    ro, b = real_buffer(pr, ctx, orc, N, H, agent)
    perms = np.zeros(n, dtype=np.uint64)
    ref.ref_ppo_permutations(4242, n, epochs, ptr(perms, U64))
    cfg = pr.PpoConfig(epochs_per_update=epochs, minibatch_size=mb, buffer_size=n)
    agent.set_ppo_mode(1)
    tc_out, tc_st = pr.ppo_update(agent, ro, cfg, 4242, perm=perms)
    agent.set_ppo_mode(0)
    simt_out, simt_st = pr.ppo_update(agent, ro, cfg, 4242, perm=perms)
    flat = agent.flatten_params()
    fo = flat.copy(); mo = np.zeros(flat.size); vo = np.zeros(flat.size); to = C.c_int64(0); so = np.zeros(4)
    offs = np.arange(N, dtype=np.uint64) * H; lens = np.full(N, H, dtype=np.uint64)
    oc = PpoCfg(0.99, 0.95, 0.2, 0.01, 0.5, epochs, mb, n, 1e-3)
    assert orc.orc_ppo_update(ptr(fo), ptr(mo), ptr(vo), C.byref(to), ptr(dims(S, 64, 64, K), SZ), 3,
                              ptr(dims(S, 64, 64, 1), SZ), 3, ptr(b["states"]), ptr(b["actions"]),
                              ptr(b["log_probs"]), ptr(b["rewards"]), ptr(b["dones"], U8), ptr(b["values"]),
                              n, S, ptr(offs, SZ), ptr(lens, SZ), ptr(b["bootstrap"]), N, C.byref(oc),
                              ptr(perms, U64), ptr(so)) == 0
    step = np.linalg.norm(fo - flat)
    d_tc = np.linalg.norm(tc_out.flatten_params() - fo) / step
    d_simt = np.linalg.norm(simt_out.flatten_params() - fo) / step
    print(f"RECORD update distance from the oracle / update size: tc {d_tc:.4f}, simt {d_simt:.4f}; policy loss "
          f"tc {tc_st.mean_policy_loss:.6g} simt {simt_st.mean_policy_loss:.6g} oracle {so[0]:.6g}")
    assert tc_st.minibatches == simt_st.minibatches == so[3] == epochs * (n // mb)
    assert tc_out.get()[3] == to.value
    assert d_tc <= 3 * d_simt + 0.05
    assert abs(tc_st.mean_policy_loss - so[0]) <= 1e-2 * (1 + abs(so[0]))
    assert abs(tc_st.mean_value_loss - so[1]) <= 1e-2 * abs(so[1])
    assert abs(tc_st.mean_entropy - so[2]) <= 1e-5 * abs(so[2])


def test_learners_equal_individual_updates(pr, ctx, orc):
    """prb_ppo_update_learners: three learners over two pods' buffers in ONE launch give exactly the
    agents (params, m, v, t) and stats that each learner's own tensor-core ppo_update gives --
    concurrency changes nothing -- and the sources are untouched (ppo.hpp:246-248)."""
    N, H, mb = 16, 128, 512
    n = N * H
    a0 = pr.Agent.init(ctx, S, K, seed=7)
    a1 = pr.Agent.init(ctx, S, K, seed=8)
    r0, _ = real_buffer(pr, ctx, orc, N, H, a0, seed=1, oracle_lp=False)
    r1, _ = real_buffer(pr, ctx, orc, N, H, a1, seed=2, oracle_lp=False)
    cfg = pr.PpoConfig(epochs_per_update=2, minibatch_size=mb, buffer_size=n)
    srcs, ros, seeds = [a0, a0, a1], [r0, r0, r1], [11, 12, 13]
    before = [a.get() for a in srcs]
    outs, stats = pr.ppo_update_learners(srcs, ros, cfg, seeds)
    for a, bf in zip(srcs, before):
        assert all(np.array_equal(x, y) for x, y in zip(a.get()[:3], bf[:3]))
    for l in range(3):
        srcs[l].set_ppo_mode(1)
        solo, st = pr.ppo_update(srcs[l], ros[l], cfg, seeds[l])
        srcs[l].set_ppo_mode(0)
        p1, m1, v1, t1 = outs[l].get()
        p2, m2, v2, t2 = solo.get()
        assert t1 == t2 == 2 * (n // mb)
        assert np.array_equal(p1, p2) and np.array_equal(m1, m2) and np.array_equal(v1, v2), l
        assert stats[l].mean_policy_loss == st.mean_policy_loss and stats[l].minibatches == st.minibatches
    assert not np.array_equal(outs[0].flatten_params(), outs[1].flatten_params())  # different seeds
    with pytest.raises(pr.UsageError):
        pr.ppo_update_learners([a0], [r0], cfg, [1], outs=[a0])  # src aliased as dst


def test_learners_beyond_one_wave(pr, ctx, orc):
    """More learners than fit on the GPU at once (8 CTAs each, 18 per wave on a B200): 20 learners
    of a 1,024-row minibatch run in two cooperative launches and each still equals its own
    tensor-core ppo_update exactly."""
    N, H, mb = 32, 64, 1024
    n = N * H
    a0 = pr.Agent.init(ctx, S, K, seed=17)
    r0, _ = real_buffer(pr, ctx, orc, N, H, a0, seed=3, oracle_lp=False)
    cfg = pr.PpoConfig(epochs_per_update=1, minibatch_size=mb, buffer_size=n)
    L = 20
    outs, stats = pr.ppo_update_learners([a0] * L, [r0] * L, cfg, list(range(100, 100 + L)))
    a0.set_ppo_mode(1)
    for l in (0, 17, 18, 19):  # both waves, and the wave boundary
        solo, st = pr.ppo_update(a0, r0, cfg, 100 + l)
        assert np.array_equal(outs[l].get()[0], solo.get()[0]), l
        assert stats[l].mean_policy_loss == st.mean_policy_loss and stats[l].minibatches == st.minibatches == n // mb
    a0.set_ppo_mode(0)
    assert len({outs[l].flatten_params().tobytes() for l in range(L)}) == L  # distinct seeds, distinct results


def test_learners_other_shapes_run_serially(pr, ctx):
    """ppo_update_learners with nets the tensor-core update does not take (PointMass 3x256): each
    learner runs its own SIMT update, results identical to ppo_update one by one."""
    N, H, mb = 64, 32, 256
    env = pr.VectorizedEnvironment.pointmass(ctx, N)
    env.reset(2)
    a0 = pr.Agent.init(ctx, 6, 2, seed=3, hidden=(256, 256, 256))
    ro = pr.Rollout.for_env(env, H)
    ro.collect(a0, env, seed=4)
    cfg = pr.PpoConfig(epochs_per_update=1, minibatch_size=mb, buffer_size=N * H)
    outs, stats = pr.ppo_update_learners([a0, a0], [ro, ro], cfg, [7, 8])
    for l, sd in enumerate((7, 8)):
        solo, st = pr.ppo_update(a0, ro, cfg, sd)
        assert np.array_equal(outs[l].get()[0], solo.get()[0]), l
        assert stats[l].minibatches == st.minibatches == (N * H) // mb
    assert not np.array_equal(outs[0].get()[0], outs[1].get()[0])


def test_tc_gate_midway_keeps_last_accepted_step(pr, ctx, orc):
    """A NaN old log-prob in the third minibatch: NumericError, and the destination holds exactly the
    state after two accepted steps -- the same as a clean 2-step update (nn.hpp:169-171)."""
    N, H, mb = 16, 64, 256
    n = N * H
    agent = pr.Agent.init(ctx, S, K, seed=9)
    agent.set_ppo_mode(1)
    ro, b = real_buffer(pr, ctx, orc, N, H, agent, oracle_lp=False)
    perm = np.random.default_rng(5).permutation(n).astype(np.uint64)
    lp = b["log_probs"].copy()
    lp[int(perm[2 * mb + 7])] = np.nan
    bad = pr.Rollout.raw(ctx, N, H, S, K)
    bad.upload(b["states"], b["actions"], lp, b["rewards"], b["dones"], b["values"], b["bootstrap"])
    cfg = pr.PpoConfig(epochs_per_update=1, minibatch_size=mb, buffer_size=n)
    out = pr.Agent(ctx, S, K)
    with pytest.raises(pr.NumericError):
        pr.ppo_update(agent, bad, cfg, 3, perm=perm, out=out)
    assert out.get()[3] == 2
    assert np.all(np.isfinite(out.flatten_params()))
    agent.set_ppo_mode(0)


def _blocks_for(S_, A):
    out, off = [], 0
    for net, n_out in (("a", A), ("c", 1)):
        d = [S_, 64, 64, n_out]
        for l in range(3):
            i, o = d[l], d[l + 1]
            out += [(f"{net}.W{l + 1}", off, off + i * o), (f"{net}.b{l + 1}", off + i * o, off + i * o + o)]
            off += i * o + o
        if net == "a":
            out.append(("log_std", off, off + A))
            off += A
    return out


@pytest.mark.parametrize("K_,mb,compact", [(3, 1024, False), (3, 700, True), (30, 700, True), (30, 1024, True),
                                           (2, 128, True)])
def test_tc_gradient_blocks_shapes(pr, ctx, orc, K_, mb, compact):
    """The tensor-core update's reduced gradient at other shapes: odd action counts (4-byte action
    copies), a partial last CTA (mb = 700: rows 640-699 live, 700-767 invalid), a single-CTA
    learner (mb = 128), and both buffer forms -- full rows (raw upload: obs_mode 0, rows at every
    4-byte shift of the 16-byte bulk-copy window) and the collected compact rows + shared-feature
    table (obs_mode 1).  Compact buffers keep the rollout's own old log-probs (the oracle gets the
    same values); full-row buffers use the oracle's.  Tolerance TOL_BLOCK per block."""
    S_ = 1 + 6 * K_
    N, H = 16, 64
    n = N * H
    m = pr.synthetic_market(K_, 2048, 2112)
    ind = pr.compute_indicators(m["high"], m["low"], m["close"])
    market = pr.MarketData(ctx, m["close"], ind)
    env = pr.VectorizedEnvironment.stock(ctx, market, pr.StockConfig(), 1500, 2047, N)
    env.reset(5)
    agent = pr.Agent.init(ctx, S_, K_, seed=9)
    agent.set_ppo_mode(1)
    ro = pr.Rollout.for_env(env, H)
    ro.collect(agent, env, seed=31)
    b = ro.download()
    flat = agent.flatten_params()
    if not compact:
        pa = sum((i + 1) * o for i, o in zip([S_, 64, 64], [64, 64, K_]))
        mean = np.zeros((n, K_))
        orc.orc_mlp_forward(ptr(np.ascontiguousarray(flat[:pa])), ptr(dims(S_, 64, 64, K_), SZ), 3,
                            ptr(np.ascontiguousarray(b["states"])), n, ptr(mean), None)
        ls = np.ascontiguousarray(flat[pa:pa + K_])
        b["log_probs"] = np.array([orc.orc_gaussian_row_log_prob(ptr(ls), K_, ptr(np.ascontiguousarray(mean[i])),
                                                                 ptr(np.ascontiguousarray(b["actions"][i])))
                                   for i in range(n)])
        ro = pr.Rollout.raw(ctx, N, H, S_, K_)
        ro.upload(b["states"], b["actions"], b["log_probs"], b["rewards"], b["dones"], b["values"], b["bootstrap"])
    perm = np.random.default_rng(4).permutation(n).astype(np.uint64)
    cfg = pr.PpoConfig(epochs_per_update=1, minibatch_size=mb, buffer_size=n - n % mb, learning_rate=0.0)
    out = pr.Agent(ctx, S_, K_)
    pr.ppo_update(agent, ro, cfg, 1, perm=perm, out=out)
    g = np.zeros(agent.param_count)
    ctx.lib.prb_debug_agent_grads(out.h, g.ctypes.data_as(C.POINTER(C.c_double)))
    # the gradient the device left is its LAST step's: minibatch n // mb - 1 of the permutation
    steps = (n - n % mb) // mb
    adv, ret = ro.buffer_advantages(cfg, normalize=True)
    idx = perm[(steps - 1) * mb:steps * mb].astype(np.int64)
    og, ol = np.zeros(flat.size), np.zeros(3)
    oc = PpoCfg(0.99, 0.95, 0.2, 0.01, 0.5, 1, mb, n - n % mb, 0.0)
    assert orc.orc_ppo_loss_grads(ptr(flat), ptr(dims(S_, 64, 64, K_), SZ), 3, ptr(dims(S_, 64, 64, 1), SZ), 3,
                                  ptr(np.ascontiguousarray(b["states"][idx])),
                                  ptr(np.ascontiguousarray(b["actions"][idx])),
                                  ptr(np.ascontiguousarray(b["log_probs"][idx])), ptr(np.ascontiguousarray(adv[idx])),
                                  ptr(np.ascontiguousarray(ret[idx])), mb, C.byref(oc), ptr(og), ptr(ol)) == 0
    errs = {}
    for name, lo, hi in _blocks_for(S_, K_):
        ref = og[lo:hi]
        errs[name] = float(np.linalg.norm(g[lo:hi] - ref) / max(np.linalg.norm(ref), 1e-30))
    print(f"RECORD tc gradient rel L2 per block K={K_} mb={mb} compact={compact}:", errs)
    assert max(errs.values()) <= TOL_BLOCK, errs
