"""GPU parity: policy, rollout, GAE, PPO loss/grads, Adam, ppo_update, fusion
and leaderboard ranking through the C ABI vs the C oracle.

Tolerances (fp32 SIMT on device vs fp64 oracle fed the SAME fp32-rounded
parameters and inputs):
  * MLP outputs / actions / values:  |d| <= 1e-5 * (1 + |x|)
  * log-probs:                       |d| <= 2e-4 (30-term fp32 sums)
  * GAE raw advantages / returns:    bit-exact fp32 (fp64 recursion on device)
  * normalised advantages:           |d| <= 1e-5 * (1 + |x|)
  * PPO gradients:                   |d| <= 1e-4 * max|g| + 1e-7
  * Adam / ppo_update params:        |d| <= 2e-6 + 1e-5|x| per step
Integer/indexing work (leaderboard order) is bit-exact.
"""
import ctypes as C

import numpy as np
import pytest

from oracle_bind import MT64, PpoCfg, StockCfg, ptr, D, I64, SZ, U8, U64

pytestmark = pytest.mark.gpu


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


def split_flat(orc, flat, S, A, hidden):
    ad = dims(S, *hidden, A)
    pa = orc.orc_mlp_param_count(ptr(ad, SZ), len(ad) - 1)
    return np.ascontiguousarray(flat[:pa]), np.ascontiguousarray(flat[pa:pa + A]), np.ascontiguousarray(flat[pa + A:])


def oracle_forward(orc, params, d, X):
    n = X.shape[0]
    Y = np.zeros((n, int(d[-1])))
    orc.orc_mlp_forward(ptr(params), ptr(d, SZ), len(d) - 1, ptr(np.ascontiguousarray(X)), n, ptr(Y), None)
    return Y


@pytest.mark.parametrize("S,A,hidden,n", [(181, 30, (64, 64), 300), (6, 2, (256, 256, 256), 100),
                                          (3, 1, (8,), 5)])
def test_policy_parity(pr, ctx, orc, S, A, hidden, n):
    flat = f32(pr.artifact_init(S, A, 7, hidden))
    rng = np.random.default_rng(S)
    agent = pr.Agent(ctx, S, A, hidden)
    # non-zero log_std so sigma != 1 matters
    actor, log_std, critic = split_flat(orc, flat, S, A, hidden)
    log_std = f32(rng.uniform(-0.5, 0.3, A))
    flat = np.concatenate([actor, log_std, critic])
    agent.set(flat)
    states = f32(rng.uniform(-2, 2, (n, S)))
    out = agent.policy_sample(states, seed=42, counter=3, with_values=True)
    mean_o = oracle_forward(orc, actor, dims(S, *hidden, A), states)
    val_o = oracle_forward(orc, critic, dims(S, *hidden, 1), states)[:, 0]
    eps = f32(out["eps"])
    act_o = np.zeros((n, A)); lp_o = np.zeros(n)
    orc.orc_policy_sample_eps(ptr(actor), ptr(dims(S, *hidden, A), SZ), len(hidden) + 1, ptr(log_std),
                              ptr(states), n, ptr(eps), ptr(act_o), ptr(lp_o))
    assert np.all(np.abs(out["actions"] - act_o) <= 1e-5 * (1 + np.abs(act_o)))
    assert np.max(np.abs(out["log_probs"] - lp_o)) <= 2e-4
    assert np.all(np.abs(out["values"] - val_o) <= 1e-5 * (1 + np.abs(val_o)))
    mean_d = agent.policy_mean(states)
    assert np.all(np.abs(mean_d - mean_o) <= 1e-5 * (1 + np.abs(mean_o)))
    # stored log-probs equal gaussian_log_prob of the sampled actions bit for bit (test_nn.cpp:274-283)
    assert np.array_equal(agent.log_prob(states, out["actions"]), out["log_probs"])
    assert np.array_equal(agent.value(states), out["values"])
    # injected-noise seam reproduces the sampled actions exactly
    again = agent.policy_sample(states, seed=0, eps=out["eps"])
    assert np.array_equal(again["actions"], out["actions"])


def test_policy_noise_stream(pr, ctx):
    S, A = 4, 30
    agent = pr.Agent.init(ctx, S, A, seed=1, hidden=(8,))
    st = np.zeros((4096, S))
    e1 = agent.policy_sample(st, seed=5, counter=0)["eps"]
    e2 = agent.policy_sample(st, seed=5, counter=0)["eps"]
    e3 = agent.policy_sample(st, seed=5, counter=1)["eps"]
    assert np.array_equal(e1, e2) and not np.array_equal(e1, e3)
    x = e1.ravel()
    assert abs(x.mean()) < 4 / np.sqrt(x.size) and abs(x.std() - 1) < 0.01
    # degenerate variance collapses to the mean (test_nn.cpp:236-247)
    flat = pr.artifact_init(S, A, 1, (8,))
    P = flat.size
    a_cnt = S * 8 + 8 + 8 * A + A
    flat[a_cnt:a_cnt + A] = -20.0
    agent.set(flat)
    rng = np.random.default_rng(0)
    s = rng.uniform(-1, 1, (6, S))
    assert np.allclose(agent.policy_sample(s, seed=9)["actions"], agent.policy_mean(s), atol=1e-6)
    bad = s.copy(); bad[2, 1] = np.nan
    with pytest.raises(pr.NumericError):
        agent.policy_sample(bad, seed=1)  # nn.hpp:252 check_finite


def _oracle_gae(orc, r, v, d, boot, N, H, gamma, lam, normalize):
    n = N * H
    offs = np.arange(N, dtype=np.uint64) * H; lens = np.full(N, H, dtype=np.uint64)
    adv = np.zeros(n); ret = np.zeros(n)
    assert orc.orc_buffer_advantages(ptr(r), ptr(v), ptr(d, U8), n, ptr(offs, SZ), ptr(lens, SZ), ptr(boot), N,
                                     gamma, lam, 1 if normalize else 0, ptr(adv), ptr(ret)) == 0
    return adv, ret


@pytest.mark.parametrize("N,H", [(1, 1), (7, 33), (300, 256), (4096, 8), (256, 100), (128, 256), (1024, 17)])
def test_gae_parity(pr, ctx, orc, N, H):
    rng = np.random.default_rng(N * 31 + H)
    n = N * H
    S, A = 2, 1
    r = f32(rng.normal(size=n) * 3); v = f32(rng.normal(size=n)); d = (rng.integers(0, 9, n) == 0).astype(np.uint8)
    boot = f32(rng.normal(size=N))
    ro = pr.Rollout.raw(ctx, N, H, S, A)
    ro.upload(np.zeros((n, S)), np.zeros((n, A)), np.zeros(n), r, d, v, boot)
    cfg = pr.PpoConfig(gamma=0.99, gae_lambda=0.95)
    raw_a, raw_r = ro.buffer_advantages(cfg, normalize=False)
    oa, orr = _oracle_gae(orc, r, v, d, boot, N, H, 0.99, 0.95, False)
    assert np.array_equal(raw_a, f32(oa)) and np.array_equal(raw_r, f32(orr))  # fp64 recursion, fp32 store
    na, nr = ro.buffer_advantages(cfg, normalize=True)
    ona, _ = _oracle_gae(orc, r, v, d, boot, N, H, 0.99, 0.95, True)
    assert np.all(np.abs(na - ona) <= 1e-5 * (1 + np.abs(ona)))
    if n > 1:
        assert abs(na.mean()) < 1e-6 and abs(na.std() - 1) < 1e-5


def test_gae_known_answers(pr, ctx):
    # test_ppo.cpp:71-75 single step; lambda=0 gives one-step TD errors (:77-95)
    ro = pr.Rollout.raw(ctx, 1, 1, 1, 1)
    ro.upload(np.zeros((1, 1)), np.zeros((1, 1)), [0.0], [0.5], [0], [2.0], [3.0])
    a, r = ro.buffer_advantages(pr.PpoConfig(gamma=0.9, gae_lambda=0.95), normalize=False)
    assert abs(a[0] - (0.5 + 0.9 * 3.0 - 2.0)) < 1e-6 and abs(r[0] - (a[0] + 2.0)) < 1e-6
    with pytest.raises(pr.UsageError):
        pr.Rollout.raw(ctx, 2, 2, 1, 1).buffer_advantages(pr.PpoConfig())  # empty buffer: coverage check


def _upload_random_buffer(pr, ctx, rng, N, H, S, A):
    n = N * H
    st = f32(rng.uniform(-1, 1, (n, S))); ac = f32(rng.normal(size=(n, A))); lp = f32(rng.uniform(-4, -1, n))
    rw = f32(rng.normal(size=n)); dn = (rng.integers(0, 10, n) == 0).astype(np.uint8); vl = f32(rng.normal(size=n))
    bt = f32(rng.normal(size=N))
    ro = pr.Rollout.raw(ctx, N, H, S, A)
    ro.upload(st, ac, lp, rw, dn, vl, bt)
    return ro, dict(states=st, actions=ac, log_probs=lp, rewards=rw, dones=dn, values=vl, bootstrap=bt)


@pytest.mark.parametrize("S,A,hidden,mb", [(11, 3, (8, 8), 37), (181, 30, (64, 64), 1024), (6, 2, (256, 256, 256), 64)])
def test_ppo_loss_grads_parity(pr, ctx, orc, S, A, hidden, mb):
    rng = np.random.default_rng(S + mb)
    N, H = 16, 64
    flat = f32(pr.artifact_init(S, A, 5, hidden))
    actor, _, critic = split_flat(orc, flat, S, A, hidden)
    flat = np.concatenate([actor, f32(rng.uniform(-0.3, 0.3, A)), critic])
    agent = pr.Agent(ctx, S, A, hidden)
    agent.set(flat)
    ro, buf = _upload_random_buffer(pr, ctx, rng, N, H, S, A)
    adv = f32(rng.normal(size=N * H)); ret = f32(rng.normal(size=N * H))
    ro.set_advantages(adv, ret)
    rows = rng.choice(N * H, size=mb, replace=False).astype(np.uint64)
    cfg = pr.PpoConfig()
    losses, g = ro.ppo_loss_grads(agent, rows, cfg)
    oc = PpoCfg(0.99, 0.95, 0.2, 0.01, 0.5, 4, mb, N * H, 1e-3)
    og = np.zeros(flat.size); ol = np.zeros(3)
    idx = rows.astype(np.int64)
    assert orc.orc_ppo_loss_grads(ptr(flat), ptr(dims(S, *hidden, A), SZ), len(hidden) + 1,
                                  ptr(dims(S, *hidden, 1), SZ), len(hidden) + 1,
                                  ptr(np.ascontiguousarray(buf["states"][idx])),
                                  ptr(np.ascontiguousarray(buf["actions"][idx])),
                                  ptr(np.ascontiguousarray(buf["log_probs"][idx])), ptr(np.ascontiguousarray(adv[idx])),
                                  ptr(np.ascontiguousarray(ret[idx])), mb, C.byref(oc), ptr(og), ptr(ol)) == 0
    assert np.all(np.abs(losses - ol) <= 1e-4 * (1 + np.abs(ol))), (losses, ol)
    scale = np.max(np.abs(og))
    assert np.max(np.abs(g - og)) <= 1e-4 * scale + 1e-7, np.max(np.abs(g - og)) / scale


def test_ppo_losses_known_answers(pr, ctx):
    S, A = 3, 2
    agent = pr.Agent.init(ctx, S, A, seed=31, hidden=(8, 8))
    rng = np.random.default_rng(5)
    n = 6
    st = f32(rng.uniform(-1, 1, (n, S))); ac = f32(rng.uniform(-1, 1, (n, A)))
    lp = agent.log_prob(st, ac).astype(np.float64)  # ratio = 1 (test_ppo.cpp:170-186)
    ro = pr.Rollout.raw(ctx, 1, n, S, A)
    ro.upload(st, ac, lp, np.zeros(n), np.zeros(n, np.uint8), np.zeros(n), [0.0])
    adv = np.array([1.0, -0.5, 0.25, 2.0, -1.5, 0.75])
    ro.set_advantages(adv, np.zeros(n))
    losses, _ = ro.ppo_loss_grads(agent, np.arange(n), pr.PpoConfig())
    assert abs(losses[0] + adv.mean()) < 1e-6
    ro.set_advantages(np.zeros(n), np.zeros(n))  # zero advantages -> zero policy loss (:188-202)
    assert ro.ppo_loss_grads(agent, np.arange(n), pr.PpoConfig())[0][0] == 0.0
    ro.set_advantages(np.full(n, np.nan), np.zeros(n))  # NonFiniteNamesComponent (:231-246)
    with pytest.raises(pr.NumericError, match="policy_loss"):
        ro.ppo_loss_grads(agent, np.arange(n), pr.PpoConfig())
    # hand-computed clipped terms (:204-229)
    ratios = np.array([0.5, 0.5, 1.5, 1.5, 1.0, 1.0])
    ro.upload(st, ac, lp - np.log(ratios), np.zeros(n), np.zeros(n, np.uint8), np.zeros(n), [0.0])
    ro.set_advantages(np.array([1.0, -2.0, 1.0, -2.0, 0.0, 0.0]), np.zeros(n))
    pl = ro.ppo_loss_grads(agent, np.arange(4), pr.PpoConfig(clip_eps=0.2))[0][0]
    assert abs(pl - (-(0.5 - 1.6 + 1.2 - 3.0) / 4.0)) < 1e-5


def test_adam_parity_and_known_answers(pr, ctx, orc):
    S, A, hid = 5, 2, (4,)
    agent = pr.Agent.init(ctx, S, A, seed=1, hidden=hid)
    P = agent.param_count
    p0 = agent.flatten_params()
    rng = np.random.default_rng(2)
    po, mo, vo, to = p0.copy(), np.zeros(P), np.zeros(P), C.c_int64(0)
    for _ in range(10):
        g = f32(rng.normal(size=P))
        agent.adam_step(g)
        orc.orc_adam_step(ptr(po), ptr(g), ptr(mo), ptr(vo), C.byref(to), P, 0.9, 0.999, 1e-8, 1e-3)
    p, m, v, t = agent.get()
    assert t == to.value == 10
    assert np.all(np.abs(p - po) <= 2e-6 + 1e-5 * np.abs(po))
    assert np.allclose(m, mo, rtol=1e-5, atol=1e-7) and np.allclose(v, vo, rtol=1e-5, atol=1e-9)
    before = agent.get()
    bad = np.zeros(P); bad[3] = np.inf
    with pytest.raises(pr.NumericError):
        agent.adam_step(bad)  # rejected before touching state (nn.hpp:169-171)
    after = agent.get()
    for x, y in zip(before[:3], after[:3]):
        assert np.array_equal(x, y)
    assert before[3] == after[3]
    a1 = pr.Agent(ctx, 1, 1, ())  # FirstStepIsSignedLearningRate (test_nn.cpp:199-208)
    for gval in (3.0, -0.7):
        a1.set(np.zeros(a1.param_count))
        a1.adam_step(np.full(a1.param_count, gval))
        assert np.allclose(a1.flatten_params(), -1e-3 * np.sign(gval), atol=1e-9)


@pytest.mark.parametrize("S,A,hid", [(5, 2, (4,)), (6, 2, (1024, 1024))])  # P = 63 and 1.06M (multi-CTA gate)
def test_adam_step_device(pr, ctx, S, A, hid):
    """prb_adam_step_device (grid-wide finite gate + Adam) == the host-gradient path, and a
    non-finite gradient anywhere leaves params/m/v/t untouched (nn.hpp:169-171)."""
    rng = np.random.default_rng(1)
    a1 = pr.Agent.init(ctx, S, A, seed=2, hidden=hid)
    a2 = a1.clone()
    for step in range(3):
        g = rng.normal(size=a1.param_count).astype(np.float32)
        a1.adam_step(g.astype(np.float64))
        dg = pr.DeviceArray.from_numpy(ctx, g)  # kept alive until the step has run
        a2.adam_step_device(dg.ptr)
    p1, m1, v1, t1 = a1.get()
    p2, m2, v2, t2 = a2.get()
    assert t1 == t2 == 3
    assert np.array_equal(p1, p2) and np.array_equal(m1, m2) and np.array_equal(v1, v2)
    g[-1] = np.nan  # the last element: only the last CTA of the check sees it
    dg = pr.DeviceArray.from_numpy(ctx, g)
    with pytest.raises(pr.NumericError):
        a2.adam_step_device(dg.ptr)
    p3, m3, v3, t3 = a2.get()
    assert t3 == 3 and np.array_equal(p3, p2) and np.array_equal(m3, m2) and np.array_equal(v3, v2)
    g[-1] = 0.5
    dg = pr.DeviceArray.from_numpy(ctx, g)
    a2.adam_step_device(dg.ptr)  # usable after the rejected step
    assert a2.get()[3] == 4


def test_ppo_update_matches_reference_permutation(pr, ctx, orc, ref):
    from oracle_bind import load_ref  # noqa: F401  (ref fixture provides the std::shuffle sequence)
    S, A, hid = 6, 2, (8, 8)
    N, H = 8, 16
    n = N * H
    rng = np.random.default_rng(10)
    flat = f32(pr.artifact_init(S, A, 9, hid))
    agent = pr.Agent(ctx, S, A, hid)
    agent.set(flat)
    ro, buf = _upload_random_buffer(pr, ctx, rng, N, H, S, A)
    epochs, mb, seed = 3, 32, 1234
    perms = np.zeros(epochs * n, dtype=np.uint64)
    ref.ref_ppo_permutations(seed, n, epochs, ptr(perms, U64))
    cfg = pr.PpoConfig(epochs_per_update=epochs, minibatch_size=mb, buffer_size=n)
    new, stats = pr.ppo_update(agent, ro, cfg, seed, perm=perms)
    # oracle on the same fp32-rounded inputs
    fo = flat.copy(); mo = np.zeros(flat.size); vo = np.zeros(flat.size); to = C.c_int64(0); so = np.zeros(4)
    offs = np.arange(N, dtype=np.uint64) * H; lens = np.full(N, H, dtype=np.uint64)
    oc = PpoCfg(0.99, 0.95, 0.2, 0.01, 0.5, epochs, mb, n, 1e-3)
    assert orc.orc_ppo_update(ptr(fo), ptr(mo), ptr(vo), C.byref(to), ptr(dims(S, *hid, A), SZ), 3,
                              ptr(dims(S, *hid, 1), SZ), 3, ptr(buf["states"]), ptr(buf["actions"]),
                              ptr(buf["log_probs"]), ptr(buf["rewards"]), ptr(buf["dones"], U8), ptr(buf["values"]),
                              n, S, ptr(offs, SZ), ptr(lens, SZ), ptr(buf["bootstrap"]), N, C.byref(oc),
                              ptr(perms, U64), ptr(so)) == 0
    p, m, v, t = new.get()
    assert t == to.value == epochs * (n // mb) and stats.minibatches == so[3]
    steps = epochs * (n // mb)
    assert np.max(np.abs(p - fo)) <= steps * 2e-5, np.max(np.abs(p - fo))
    assert abs(stats.mean_policy_loss - so[0]) <= 1e-4 * (1 + abs(so[0]))
    assert abs(stats.mean_value_loss - so[1]) <= 1e-4 * (1 + abs(so[1]))
    assert abs(stats.mean_entropy - so[2]) <= 1e-5 * (1 + abs(so[2]))
    # purity: the input agent is untouched (ppo.hpp:246-248)
    assert np.array_equal(agent.flatten_params(), flat)


def test_ppo_update_properties(pr, ctx):
    S, A, hid = 1, 1, (8, 8)
    N, H = 4, 16
    rng = np.random.default_rng(3)
    agent = pr.Agent.init(ctx, S, A, seed=35, hidden=hid)
    ro, _ = _upload_random_buffer(pr, ctx, rng, N, H, S, A)
    # zero learning rate leaves params (test_ppo.cpp:248-257)
    new, _ = pr.ppo_update(agent, ro, pr.PpoConfig(buffer_size=64, minibatch_size=32, learning_rate=0.0), 7)
    assert np.array_equal(new.flatten_params(), agent.flatten_params())
    # deterministic under a fixed seed, with device-generated permutations (:259-269)
    cfg = pr.PpoConfig(buffer_size=64, minibatch_size=16)
    r1, s1 = pr.ppo_update(agent, ro, cfg, 11)
    r2, s2 = pr.ppo_update(agent, ro, cfg, 11)
    assert np.array_equal(r1.flatten_params(), r2.flatten_params()) and s1.mean_policy_loss == s2.mean_policy_loss
    r3, _ = pr.ppo_update(agent, ro, cfg, 12)
    assert not np.array_equal(r1.flatten_params(), r3.flatten_params())
    assert s1.minibatches == 4 * 4
    # one minibatch == whole buffer: device permutation and identity permutation see the same rows
    cfg1 = pr.PpoConfig(buffer_size=64, minibatch_size=64, epochs_per_update=1)
    a1, _ = pr.ppo_update(agent, ro, cfg1, 5)
    a2, _ = pr.ppo_update(agent, ro, cfg1, 5, perm=np.arange(64, dtype=np.uint64))
    assert np.allclose(a1.flatten_params(), a2.flatten_params(), atol=1e-6)
    with pytest.raises(pr.ConfigError):
        pr.ppo_update(agent, ro, pr.PpoConfig(buffer_size=64, minibatch_size=128), 1)
    with pytest.raises(pr.UsageError):
        pr.ppo_update(agent, pr.Rollout.raw(ctx, N, H, S, A), cfg, 1)  # buffer must be full (:281-289)


@pytest.mark.parametrize("S,A,hid,N,H,mb,epochs", [(181, 30, (64, 64), 64, 64, 1024, 2),
                                                    (6, 2, (256, 256, 256), 16, 32, 256, 1),
                                                    (11, 3, (8, 8), 9, 13, 37, 3)])
def test_ppo_update_persistent_equals_per_kernel_path(pr, ctx, S, A, hid, N, H, mb, epochs):
    """The persistent cooperative update (one launch, grid barriers between phases) runs the
    per-kernel path's device functions in the same reduction orders: bit-identical results."""
    rng = np.random.default_rng(S + mb)
    agent = pr.Agent.init(ctx, S, A, seed=3, hidden=hid)
    ro, _ = _upload_random_buffer(pr, ctx, rng, N, H, S, A)
    cfg = pr.PpoConfig(epochs_per_update=epochs, minibatch_size=mb, buffer_size=N * H)
    a1, s1 = pr.ppo_update(agent, ro, cfg, 21)
    pr.set_debug_option(pr.OPT_PPO_PER_KERNEL, 1)
    try:
        a2, s2 = pr.ppo_update(agent, ro, cfg, 21)
    finally:
        pr.set_debug_option(pr.OPT_PPO_PER_KERNEL, 0)
    p1, m1, v1, t1 = a1.get()
    p2, m2, v2, t2 = a2.get()
    assert t1 == t2 == epochs * ((N * H) // mb) and s1.minibatches == s2.minibatches == t1
    assert np.array_equal(p1, p2) and np.array_equal(m1, m2) and np.array_equal(v1, v2)
    assert s1.mean_policy_loss == s2.mean_policy_loss and s1.mean_value_loss == s2.mean_value_loss
    assert s1.mean_entropy == s2.mean_entropy


def test_ppo_update_nonfinite_gate_leaves_state(pr, ctx):
    """A non-finite loss aborts the update at the first step in both paths and names the
    component (ppo.hpp:169-171); the returned error leaves the source agent untouched."""
    S, A, hid, N, H = 6, 2, (8, 8), 8, 16
    rng = np.random.default_rng(4)
    agent = pr.Agent.init(ctx, S, A, seed=5, hidden=hid)
    ro, buf = _upload_random_buffer(pr, ctx, rng, N, H, S, A)
    bad = buf["rewards"].copy(); bad[5] = np.inf
    ro.upload(buf["states"], buf["actions"], buf["log_probs"], bad, buf["dones"], buf["values"], buf["bootstrap"])
    cfg = pr.PpoConfig(epochs_per_update=2, minibatch_size=32, buffer_size=N * H)
    before = agent.flatten_params().copy()
    with pytest.raises(pr.NumericError):
        pr.ppo_update(agent, ro, cfg, 3)
    assert np.array_equal(agent.flatten_params(), before)
    # the agent and the context stay usable afterwards
    ro.upload(buf["states"], buf["actions"], buf["log_probs"], buf["rewards"], buf["dones"], buf["values"],
              buf["bootstrap"])
    new, st = pr.ppo_update(agent, ro, cfg, 3)
    assert st.minibatches == 2 * (N * H // 32) and np.all(np.isfinite(new.flatten_params()))


def test_fuse_parity(pr, ctx, orc):
    S, A, hid = 5, 2, (4,)
    rng = np.random.default_rng(12)
    L = 3
    agents = []
    ps, ms, vs, ts = [], [], [], np.array([5, 9, 7], dtype=np.int64)
    for i in range(L):
        a = pr.Agent(ctx, S, A, hid)
        p = f32(rng.normal(size=a.param_count)); m = f32(rng.normal(size=a.param_count))
        v = f32(rng.uniform(0, 1, a.param_count))
        a.set(p, m, v, int(ts[i]))
        agents.append(a); ps.append(p); ms.append(m); vs.append(v)
    fused = pr.fuse_parameters(agents)
    P = agents[0].param_count
    arr = lambda xs: (D * L)(*[ptr(x) for x in xs])
    o = [np.zeros(P) for _ in range(3)]; ot = C.c_int64()
    orc.orc_fuse(arr(ps), arr(ms), arr(vs), ptr(ts, I64), L, P, ptr(o[0]), ptr(o[1]), ptr(o[2]), C.byref(ot))
    got = fused.get()
    for x, y in zip(got[:3], o):
        assert np.allclose(x, y, rtol=1e-6, atol=1e-7)
    assert got[3] == ot.value == 9
    single = pr.fuse_parameters(agents[:1])  # a single artifact is returned unchanged (pod.hpp:143)
    assert all(np.array_equal(x, y) for x, y in zip(single.get()[:3], agents[0].get()[:3]))
    with pytest.raises(pr.UsageError):
        pr.fuse_parameters([agents[0], pr.Agent(ctx, S, A, (5,))])
    # the output may be one of the inputs (the elementwise mean reads every input before writing)
    aliased = pr.fuse_parameters(agents, out=agents[1])
    assert all(np.array_equal(x, y) for x, y in zip(aliased.get()[:3], got[:3])) and aliased.get()[3] == 9


def test_leaderboard_rank_matches_sequential_insertion(pr, ctx, orc):
    rng = np.random.default_rng(31)
    for trial in range(200):
        cap = int(1 + rng.integers(0, 6)); n = int(1 + rng.integers(0, 30))
        scores = rng.uniform(-5, 5, n) if trial % 2 == 0 else rng.integers(0, 9, n).astype(np.float64)
        order = pr.leaderboard_rank(ctx, scores, np.arange(n, dtype=np.uint64), cap)
        bs = np.zeros(cap); bq = np.zeros(cap, dtype=np.uint64); bi = np.zeros(cap, dtype=np.int64)
        size = C.c_size_t(0); seq = C.c_uint64(0)
        for i, s in enumerate(scores):
            orc.orc_leaderboard_update(ptr(bs), ptr(bq, U64), ptr(bi, I64), C.byref(size), cap, C.byref(seq), float(s), i)
        assert np.array_equal(order, bi[:size.value])
    with pytest.raises(pr.NumericError):
        pr.leaderboard_rank(ctx, [1.0, np.nan], [0, 1], 2)


def _replay_stock(orc, close, ind, cfg, start, end, N, H, acts, K):
    S = 1 + 6 * K
    c = StockCfg(cfg.initial_capital, cfg.max_trade_shares, cfg.cost_rate)
    bal = np.zeros(N); sh = np.zeros(N * K); t = np.zeros(N, dtype=np.uint64); sc = np.zeros(N, dtype=np.uint64)
    er = np.zeros(N)
    orc.orc_stock_vec_reset(N, K, C.byref(c), start, ptr(bal), ptr(sh), ptr(t, SZ), ptr(sc, SZ), ptr(er))
    states = np.zeros((N, H, S)); rewards = np.zeros((N, H)); dones = np.zeros((N, H), np.uint8)
    obs = np.zeros((N, S))
    for e in range(N):
        orc.orc_stock_observation(bal[e], ptr(np.ascontiguousarray(sh[e * K:(e + 1) * K])), int(t[e]), ptr(close),
                                  ptr(ind), close.shape[1], K, C.byref(c), start, ptr(obs[e]))
    for h in range(H):
        states[:, h] = obs
        nx = np.zeros((N, S)); r = np.zeros(N); d = np.zeros(N, np.uint8)
        orc.orc_stock_vec_step(N, K, C.byref(c), start, end, ptr(close), ptr(ind), close.shape[1], ptr(bal), ptr(sh),
                               ptr(t, SZ), ptr(sc, SZ), ptr(er), ptr(np.ascontiguousarray(acts[:, h])), ptr(nx),
                               ptr(r), ptr(d, U8), ptr(np.zeros((N, S))), ptr(np.zeros(N)), ptr(np.zeros(N, np.uint64), U64))
        rewards[:, h] = r; dones[:, h] = d; obs = nx
    return states.reshape(N * H, S), rewards.ravel(), dones.ravel(), obs


@pytest.mark.parametrize("fused,K,N,H", [(0, 30, 96, 48), (1, 30, 96, 48), (2, 30, 96, 48),
                                         (2, 30, 1, 3), (2, 30, 300, 12), (2, 3, 200, 33), (1, 3, 130, 31)])
def test_collect_stock_rollout_replays_on_oracle(pr, ctx, orc, fused, K, N, H):
    """Ragged shapes too: a single env, N not a multiple of the 128-env tile, a
    small-K instantiation of the tcgen05 kernel, horizons shorter than an episode."""
    T = 200
    m = pr.synthetic_market(K, T, seed=2112)
    ind = pr.compute_indicators(m["high"], m["low"], m["close"])
    market = pr.MarketData(ctx, m["close"], ind)
    cfg = pr.StockConfig()
    start, end = 10, 40  # episodes of 30 steps inside a 48-step horizon
    env = pr.VectorizedEnvironment.stock(ctx, market, cfg, start, end, N)
    env.reset(1)
    S = 1 + 6 * K
    agent = pr.Agent.init(ctx, S, K, seed=7)
    ro = pr.Rollout.for_env(env, H)
    ro.set_mode(fused)
    ro.collect(agent, env, seed=99)
    b = ro.download()
    acts = b["actions"].reshape(N, H, K)
    st, rw, dn, final = _replay_stock(orc, np.ascontiguousarray(m["close"]), np.ascontiguousarray(ind), cfg, start,
                                      end, N, H, acts, K)
    assert np.array_equal(b["states"], f32(st))  # compact rows + shared features == full obs
    assert np.array_equal(b["rewards"], f32(rw)) and np.array_equal(b["dones"], dn)
    if H > 29:
        assert dn.reshape(N, H)[:, 29].all()
    assert np.array_equal(env.states(), f32(final))
    lp, val, boot = (agent.log_prob(b["states"], b["actions"]), agent.value(b["states"]),
                     agent.value(env.states()))
    if not fused:  # the per-step path runs exactly the standalone policy kernel
        assert np.array_equal(lp, b["log_probs"].astype(np.float32))
        assert np.array_equal(val, b["values"].astype(np.float32))
        assert np.array_equal(boot, b["bootstrap"].astype(np.float32))
    else:
        # mode 1: fused fp32 kernel, shared-feature term summed separately (fp32 order only)
        # mode 2: tcgen05 layers, bf16 operands + tanh.approx: the stated bf16 tolerance
        tl, tv = (2e-4, 1e-5) if fused == 1 else (1e-2, 5e-2)
        mean = agent.policy_mean(b["states"])
        flat = agent.flatten_params()
        ls = flat[S * 64 + 64 + 64 * 64 + 64 + 64 * K + K:][:K]
        eps = (b["actions"] - mean) / np.exp(ls)
        if fused == 1:
            lp_tol = tl * (1 + np.abs(lp))
        else:
            # bf16 path: the log-prob error is the stated mean tolerance (tv in the units of the
            # mean) propagated through log pi = sum_d(-0.5 z_d^2 + const): a mean error delta_d
            # (in sigma units) moves log pi by up to delta_d (|z_d| + delta_d / 2); plus fp32 slack
            dlt = tv * (1 + np.abs(mean)) / np.exp(ls)
            lp_tol = np.sum(dlt * (np.abs(eps) + dlt / 2), axis=1) + 1e-3 * (1 + np.abs(lp))
        assert np.all(np.abs(lp - b["log_probs"]) <= lp_tol), np.max(np.abs(lp - b["log_probs"]) / lp_tol)
        assert np.all(np.abs(val - b["values"]) <= tv * (1 + np.abs(val))), np.max(np.abs(val - b["values"]))
        assert np.all(np.abs(boot - b["bootstrap"]) <= tv * (1 + np.abs(boot)))
        # noise stream identical to the standalone sampler: eps recovered from the actions
        s0 = np.ascontiguousarray(b["states"].reshape(N, H, S)[:, 0])  # step 0 of every env
        ref_eps = agent.policy_sample(s0, seed=99, counter=0)["eps"]
        assert np.allclose(eps.reshape(N, H, K)[:, 0], ref_eps, atol=1e-3 if fused == 1 else 5e-2)


@pytest.mark.parametrize("mode,N,H", [(0, 64, 250), (2, 64, 250), (2, 1000, 40), (2, 40000, 6), (2, 1, 3)])
def test_collect_pointmass_rollout(pr, ctx, orc, mode, N, H):
    """PointMass2D worker_collect: the env transitions replay bit-exactly on the
    oracle from the recorded actions; mode 2 (tcgen05 3x256, bf16 operands)
    log-probs / values agree with the fp32 policy on the recorded states within
    the bf16 tolerance.  N=40000 spans more tiles than SMs (persistent loop)."""
    env = pr.VectorizedEnvironment.pointmass(ctx, N)
    env.reset(3)
    oracle_g = (MT64 * N)()
    st = np.zeros((N, 6)); sc = np.zeros(N, np.uint64); er = np.zeros(N)
    orc.orc_pm_vec_reset(N, 3, oracle_g, ptr(st), ptr(sc, U64), ptr(er))
    agent = pr.Agent.init(ctx, 6, 2, seed=4, hidden=(256, 256, 256))
    ro = pr.Rollout.for_env(env, H)
    ro.set_mode(mode)
    ro.collect(agent, env, seed=8)
    b = ro.download()
    states = b["states"].reshape(N, H, 6); acts = b["actions"].reshape(N, H, 2)
    for h in range(H):
        assert np.array_equal(states[:, h], f32(st)), h
        r = np.zeros(N); d = np.zeros(N, np.uint8)
        orc.orc_pm_vec_step(N, oracle_g, ptr(st), ptr(sc, U64), ptr(er), ptr(np.ascontiguousarray(acts[:, h])), ptr(r),
                            ptr(d, U8), ptr(np.zeros((N, 6))), ptr(np.zeros(N)), ptr(np.zeros(N, np.uint64), U64))
        assert np.array_equal(b["rewards"].reshape(N, H)[:, h], f32(r))
        assert np.array_equal(b["dones"].reshape(N, H)[:, h], d)
    assert np.array_equal(env.states(), f32(st))
    assert np.array_equal(env.step_counts(), sc)
    if H >= 200:
        assert b["dones"].sum() >= N
    lp, val, boot = (agent.log_prob(b["states"], b["actions"]), agent.value(b["states"]),
                     agent.value(env.states()))
    if mode == 0:
        assert np.array_equal(lp, b["log_probs"].astype(np.float32))
        assert np.array_equal(val, b["values"].astype(np.float32))
    else:  # bf16 operands + tanh.approx through 3 hidden layers of 256
        tl, tv = 1e-2, 2e-2
        assert np.all(np.abs(lp - b["log_probs"]) <= tl * (1 + np.abs(lp))), np.max(np.abs(lp - b["log_probs"]))
        assert np.all(np.abs(val - b["values"]) <= tv * (1 + np.abs(val))), np.max(np.abs(val - b["values"]))
        assert np.all(np.abs(boot - b["bootstrap"]) <= tv * (1 + np.abs(boot)))
        mean = agent.policy_mean(b["states"])
        # noise stream identical to the standalone sampler: eps recovered from the actions
        ls = _pm_log_std(agent)
        eps = (b["actions"] - mean) / np.exp(ls)
        s0 = np.ascontiguousarray(states[:, 0])
        ref_eps = agent.policy_sample(s0, seed=8, counter=0)["eps"]
        assert np.allclose(eps.reshape(N, H, 2)[:, 0], ref_eps, atol=5e-2)


def _pm_log_std(agent):
    flat = agent.flatten_params()
    pa = 6 * 256 + 256 + 2 * (256 * 256 + 256) + 256 * 2 + 2
    return flat[pa:pa + 2]


@pytest.fixture
def debug_option(pr):
    """Sets a test-only switch (PRB_OPT_* in include/prb.h) for one test and clears it after."""
    set_ = []

    def _set(opt, val=1):
        pr.set_debug_option(opt, val)
        set_.append(opt)
    yield _set
    for o in set_:
        pr.set_debug_option(o, 0)


@pytest.mark.parametrize("N,H", [(64, 250), (1000, 40), (40000, 6)])
def test_collect_pointmass_cta_pair_kernel(pr, ctx, orc, debug_option, N, H):
    """The opt-in CTA-pair (cta_group::2) PointMass kernel (PRB_OPT_PM_CTA_PAIR) passes the same
    replay / tolerance checks as the default kernel."""
    debug_option(pr.OPT_PM_CTA_PAIR)
    test_collect_pointmass_rollout(pr, ctx, orc, 2, N, H)


@pytest.mark.parametrize("K,N,H", [(30, 96, 48), (30, 300, 17), (3, 200, 40)])
def test_collect_stock_tc_redo_path(pr, ctx, orc, debug_option, K, N, H):
    """The tcgen05 stock rollout's rare redo path (a buy quantity outside the division-free
    certificate -> the warp redoes the step's trades with the reference's division) forced on
    every step (PRB_OPT_TC_FORCE_REDO): the env transitions still replay bit-exactly on the
    oracle."""
    debug_option(pr.OPT_TC_FORCE_REDO)
    test_collect_stock_rollout_replays_on_oracle(pr, ctx, orc, 2, K, N, H)


@pytest.mark.parametrize("max_trade,cost,cap", [(37.5, 0.002, 1e6), (1000.0, 0.0, 2e4), (3.0, 0.01, 5e5)])
def test_collect_stock_tc_config_variants(pr, ctx, orc, max_trade, cost, cap):
    """The tcgen05 stock rollout under other StockConfigs, replayed bit-exactly on the oracle:
    a non-integer max_trade_shares (the fp64 desired-quantity path instead of the exact fp32
    one), a cash-starved portfolio with large trades and no cost (most buys cash-limited: the
    division-free certificate on almost every buy), and tiny trades with a high cost rate."""
    K, N, H, T = 30, 256, 40, 200
    m = pr.synthetic_market(K, T, seed=2112)
    ind = pr.compute_indicators(m["high"], m["low"], m["close"])
    market = pr.MarketData(ctx, m["close"], ind)
    cfg = pr.StockConfig(initial_capital=cap, max_trade_shares=max_trade, cost_rate=cost)
    start, end = 10, 40
    env = pr.VectorizedEnvironment.stock(ctx, market, cfg, start, end, N)
    env.reset(1)
    agent = pr.Agent.init(ctx, 1 + 6 * K, K, seed=7)
    ro = pr.Rollout.for_env(env, H)
    ro.set_mode(2)
    ro.collect(agent, env, seed=5)
    b = ro.download()
    acts = b["actions"].reshape(N, H, K)
    st, rw, dn, final = _replay_stock(orc, np.ascontiguousarray(m["close"]), np.ascontiguousarray(ind), cfg, start,
                                      end, N, H, acts, K)
    assert np.array_equal(b["states"], f32(st))
    assert np.array_equal(b["rewards"], f32(rw)) and np.array_equal(b["dones"], dn)
    assert np.array_equal(env.states(), f32(final))


@pytest.mark.parametrize("hid", [(64, 64), (8, 8)])
def test_ppo_update_gate_midway_rolls_back(pr, ctx, hid, debug_option):
    """A non-finite loss at a LATER minibatch step (a NaN old log-prob placed in epoch 0's third
    minibatch by an injected permutation): the persistent update stores each Adam step before
    its gate is known and undoes it on failure, so the destination agent holds exactly the state
    after the last accepted step -- params, m, v and t identical to the per-kernel path, whose
    Adam kernel runs only after the gate (adam_step nn.hpp:169-171)."""
    S, A, N, H, mb = 181, 30, 64, 64, 512
    n = N * H
    rng = np.random.default_rng(11)
    agent = pr.Agent.init(ctx, S, A, seed=9, hidden=hid)
    ro, buf = _upload_random_buffer(pr, ctx, rng, N, H, S, A)
    bad_row = 1234
    lp = buf["log_probs"].copy()
    lp[bad_row] = np.nan
    ro.upload(buf["states"], buf["actions"], lp, buf["rewards"], buf["dones"], buf["values"], buf["bootstrap"])
    perm = np.concatenate([rng.permutation(n) for _ in range(2)]).astype(np.uint64)
    k = int(np.where(perm[:n] == bad_row)[0][0])
    perm[[k, 2 * mb + 5]] = perm[[2 * mb + 5, k]]  # the bad row lands in step 2
    cfg = pr.PpoConfig(epochs_per_update=2, minibatch_size=mb, buffer_size=n)
    outs = []
    for graph in (False, True):
        if graph:
            debug_option(pr.OPT_PPO_PER_KERNEL)
        out = pr.Agent.init(ctx, S, A, seed=1, hidden=hid)
        with pytest.raises(pr.NumericError):
            pr.ppo_update(agent, ro, cfg, 3, perm=perm, out=out)
        outs.append(out.get())
    (p1, m1, v1, t1), (p2, m2, v2, t2) = outs
    t0 = agent.get()[3]
    assert t1 == t2 == t0 + 2
    assert np.array_equal(p1, p2) and np.array_equal(m1, m2) and np.array_equal(v1, v2)
    assert not np.array_equal(p1, agent.flatten_params())  # two steps were applied
