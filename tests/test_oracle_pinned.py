"""Pin the C restatement (oracle/liboracle.so) against the reference itself
(oracle/_ref/libpodracer_ref_exact.so, the unmodified headers behind a shim,
same -ffp-contract=off flags) and against the known answers the reference's
own unit tests hold (file:line cited per test).  CPU only."""
import ctypes as C

import numpy as np
import pytest

from oracle_bind import (MT64, PpoCfg, StockCfg, derive_seed, indicators, ptr, synthetic_market_np, D, I64, SZ,
                         U64, U8)


def test_derive_seed_matches_reference(orc, ref):
    rng = np.random.default_rng(0)
    for _ in range(200):
        base = int(rng.integers(0, 2**63))
        tags = [int(x) for x in rng.integers(0, 2**40, size=int(rng.integers(0, 4)))]
        assert derive_seed(orc, base, *tags) == derive_seed(ref, base, *tags)


def test_mt19937_64_and_uniform_real_match_libstdcxx(orc, ref):
    for seed in [0, 1, 5489, 2**63 + 7, 123456789]:
        g = MT64()
        orc.orc_mt64_seed(C.byref(g), seed)
        got = np.array([orc.orc_mt64_next(C.byref(g)) for _ in range(700)], dtype=np.uint64)
        exp = np.zeros(700, dtype=np.uint64)
        ref.ref_mt64_draws(seed, 700, ptr(exp, U64))
        assert np.array_equal(got, exp)
        g = MT64()
        orc.orc_mt64_seed(C.byref(g), seed)
        got = np.array([orc.orc_uniform_real(C.byref(g), -0.4, 0.4) for _ in range(700)])
        exp = np.zeros(700)
        ref.ref_uniform_real_draws(seed, -0.4, 0.4, 700, ptr(exp))
        assert np.array_equal(got, exp)  # bit-exact


def _stock_step(lib, fn, bal, sh, t, act, close, cfg):
    K = close.shape[0]
    bal_c = C.c_double(bal)
    sh = np.ascontiguousarray(sh, dtype=np.float64).copy()
    t_c = C.c_size_t(t)
    r = C.c_double()
    d = C.c_int()
    act = np.ascontiguousarray(act, dtype=np.float64)
    if fn == "orc":
        c = StockCfg(*cfg)
        rc = lib.orc_stock_env_step(C.byref(bal_c), ptr(sh), C.byref(t_c), ptr(act), ptr(close), close.shape[1], K,
                                    C.byref(c), C.byref(r), C.byref(d))
    else:
        c3 = np.array(cfg, dtype=np.float64)
        rc = lib.ref_stock_env_step(C.byref(bal_c), ptr(sh), C.byref(t_c), ptr(act), ptr(close), close.shape[1], K,
                                    ptr(c3), C.byref(r), C.byref(d))
    return rc, bal_c.value, sh, t_c.value, r.value, d.value


def test_stock_step_known_answers(orc):
    # test_stock_env.cpp:84-107 HandAccountingWithCost: 1000 -> 499 after buying 50 @10 with 0.2% cost
    close = np.full((1, 3), 10.0)
    rc, bal, sh, t, r, d = _stock_step(orc, "orc", 1000.0, [0.0], 0, [0.5], close, (1000.0, 100.0, 0.002))
    assert rc == 0 and sh[0] == 50.0 and abs(bal - 499.0) < 1e-12 and abs(r - (-1.0)) < 1e-12
    # test_stock_env.cpp:124-144 BuysClippedToAffordableBalance -> 9 shares
    close = np.full((1, 3), 100.0)
    rc, bal, sh, t, r, d = _stock_step(orc, "orc", 1000.0, [0.0], 0, [1.0], close, (1000.0, 1000.0, 0.002))
    assert sh[0] == 9.0 and bal >= 0.0
    # test_stock_env.cpp:60-82 RoundTripAtConstantPriceIsLossless
    close = np.full((1, 40), 10.0)
    rc, bal, sh, t, r1, d = _stock_step(orc, "orc", 1000.0, [0.0], 0, [1.0], close, (1000.0, 50.0, 0.0))
    assert sh[0] == 50.0
    rc, bal, sh, t, r2, d = _stock_step(orc, "orc", bal, sh, t, [-1.0], close, (1000.0, 50.0, 0.0))
    assert sh[0] == 0.0 and abs(bal - 1000.0) < 1e-12 and abs(r1 + r2) < 1e-12
    # stock_env.hpp:64-66: stepping at the last row is a UsageError
    rc, *_ = _stock_step(orc, "orc", 1000.0, [0.0], 2, [0.0], np.full((1, 3), 10.0), (1000.0, 100.0, 0.002))
    assert rc == 3


def test_stock_step_random_sequences_bit_exact(orc, ref):
    rng = np.random.default_rng(7)
    close, high, low = synthetic_market_np(5, 120, seed=3)
    for trial in range(30):
        cfg = (float(rng.choice([1e3, 1e5, 1e6])), float(rng.choice([10.0, 100.0])), float(rng.choice([0.0, 0.002])))
        s_o = s_r = None
        bal_o = bal_r = cfg[0]
        sh_o = sh_r = np.zeros(5)
        t_o = t_r = 0
        while t_o + 1 < close.shape[1]:
            a = rng.uniform(-1.5, 1.5, size=5)
            o = _stock_step(orc, "orc", bal_o, sh_o, t_o, a, close, cfg)
            f = _stock_step(ref, "ref", bal_r, sh_r, t_r, a, close, cfg)
            assert o[0] == f[0] == 0
            assert o[1] == f[1] and np.array_equal(o[2], f[2]) and o[3] == f[3] and o[4] == f[4] and o[5] == f[5]
            _, bal_o, sh_o, t_o, _, _ = o
            _, bal_r, sh_r, t_r, _, _ = f
            assert bal_o >= 0 and np.all(sh_o >= 0) and np.all(sh_o == np.trunc(sh_o))  # :165-181 feasibility


def test_indicators_bit_exact(orc, ref):
    close, high, low = synthetic_market_np(4, 300, seed=11)
    a = indicators(orc, high, low, close)
    b = indicators(ref, high, low, close)
    assert np.array_equal(a, b)


def _stock_vec_orc(orc, close, ind, cfg, start, end, N, actions_seq):
    K, T = close.shape
    S = 1 + 6 * K
    c = StockCfg(*cfg)
    bal = np.zeros(N); sh = np.zeros(N * K); t = np.zeros(N, dtype=np.uint64); sc = np.zeros(N, dtype=np.uint64)
    ret = np.zeros(N)
    orc.orc_stock_vec_reset(N, K, C.byref(c), start, ptr(bal), ptr(sh), ptr(t, SZ), ptr(sc, SZ), ptr(ret))
    outs = []
    for acts in actions_seq:
        nxt = np.zeros((N, S)); r = np.zeros(N); d = np.zeros(N, dtype=np.uint8); term = np.zeros((N, S))
        tr = np.zeros(N); tl = np.zeros(N, dtype=np.uint64)
        rc = orc.orc_stock_vec_step(N, K, C.byref(c), start, end, ptr(close), ptr(ind), T, ptr(bal), ptr(sh),
                                    ptr(t, SZ), ptr(sc, SZ), ptr(ret), ptr(np.ascontiguousarray(acts)), ptr(nxt),
                                    ptr(r), ptr(d, U8), ptr(term), ptr(tr), ptr(tl, U64))
        assert rc == 0
        outs.append((nxt, r, d, term, tr, tl))
    return outs


def test_stock_vecenv_with_auto_reset_bit_exact(orc, ref):
    K, T, N = 3, 80, 6
    close, high, low = synthetic_market_np(K, T, seed=5)
    ind = indicators(orc, high, low, close)
    cfg = (1e4, 100.0, 0.002)
    start, end = 40, 52  # 12-step episodes -> several auto-resets
    rng = np.random.default_rng(1)
    seq = [rng.uniform(-1.2, 1.2, size=(N, K)) for _ in range(30)]
    got = _stock_vec_orc(orc, close, ind, cfg, start, end, N, seq)
    h = ref.ref_stock_vec_create(ptr(close), ptr(ind), T, K, ptr(np.array(cfg)), start, end, N)
    S = 1 + 6 * K
    obs0 = np.zeros((N, S))
    assert ref.ref_vec_reset(h, 9, ptr(obs0)) == 0
    for (nxt, r, d, term, tr, tl), acts in zip(got, seq):
        e_nxt = np.zeros((N, S)); e_r = np.zeros(N); e_d = np.zeros(N, dtype=np.uint8); e_term = np.zeros((N, S))
        e_tr = np.zeros(N); e_tl = np.zeros(N, dtype=np.uint64)
        assert ref.ref_vec_step(h, ptr(np.ascontiguousarray(acts)), K, ptr(e_nxt), ptr(e_r), ptr(e_d, U8),
                                ptr(e_term), ptr(e_tr), ptr(e_tl, U64)) == 0
        assert np.array_equal(nxt, e_nxt) and np.array_equal(r, e_r) and np.array_equal(d, e_d)
        m = d.astype(bool)
        assert np.array_equal(term[m], e_term[m]) and np.array_equal(tr[m], e_tr[m]) and np.array_equal(tl[m], e_tl[m])
    assert any(o[2].any() for o in got)
    ref.ref_vec_destroy(h)


def test_pointmass_known_answers(orc):
    s = np.array([0.3, -0.2, 0.0, 0.0, 0.3, -0.2]); a = np.zeros(2); out = np.zeros(6)
    r = C.c_double(); d = C.c_int()
    orc.orc_pointmass_step(ptr(s), ptr(a), 0, ptr(out), C.byref(r), C.byref(d))  # test_envs.cpp:62-67
    assert d.value == 1 and abs(r.value - 10.0) < 1e-15
    s = np.array([0.9, 0.9, 0.0, 0.0, -0.9, -0.9])  # test_envs.cpp:95-99 StepLimitAt200
    orc.orc_pointmass_step(ptr(s), ptr(a), 198, ptr(out), C.byref(r), C.byref(d)); assert d.value == 0
    orc.orc_pointmass_step(ptr(s), ptr(a), 199, ptr(out), C.byref(r), C.byref(d)); assert d.value == 1


def test_pointmass_vecenv_reset_and_steps_bit_exact(orc, ref):
    N = 16
    gens = (MT64 * N)()
    st = np.zeros((N, 6)); sc = np.zeros(N, dtype=np.uint64); er = np.zeros(N)
    orc.orc_pm_vec_reset(N, 77, gens, ptr(st), ptr(sc, U64), ptr(er))
    h = ref.ref_pm_vec_create(N)
    e0 = np.zeros((N, 6))
    ref.ref_vec_reset(h, 77, ptr(e0))
    assert np.array_equal(st, e0)  # test_envs.cpp:114-121 SingleEnvMatchesDerivedStream, for every row
    rng = np.random.default_rng(5)
    resets = 0
    for _ in range(400):
        acts = np.ascontiguousarray(rng.uniform(-1.3, 1.3, size=(N, 2)))
        r = np.zeros(N); d = np.zeros(N, dtype=np.uint8); term = np.zeros((N, 6)); tr = np.zeros(N)
        tl = np.zeros(N, dtype=np.uint64)
        orc.orc_pm_vec_step(N, gens, ptr(st), ptr(sc, U64), ptr(er), ptr(acts), ptr(r), ptr(d, U8), ptr(term),
                            ptr(tr), ptr(tl, U64))
        e_nxt = np.zeros((N, 6)); e_r = np.zeros(N); e_d = np.zeros(N, dtype=np.uint8); e_term = np.zeros((N, 6))
        e_tr = np.zeros(N); e_tl = np.zeros(N, dtype=np.uint64)
        ref.ref_vec_step(h, ptr(acts), 2, ptr(e_nxt), ptr(e_r), ptr(e_d, U8), ptr(e_term), ptr(e_tr), ptr(e_tl, U64))
        assert np.array_equal(st, e_nxt) and np.array_equal(r, e_r) and np.array_equal(d, e_d)
        m = d.astype(bool)
        resets += int(m.sum())
        assert np.array_equal(term[m], e_term[m]) and np.array_equal(tl[m], e_tl[m]) and np.array_equal(tr[m], e_tr[m])
    assert resets >= N  # the 200-step limit alone forces every row through a reset
    ref.ref_vec_destroy(h)


def _dims(*d):
    return np.array(d, dtype=np.uint64)


def _flat_init(ref, S, A, seed, hidden):
    h = np.array(hidden, dtype=np.uint64)
    P = ref.ref_artifact_init(S, A, seed, 1e-3, ptr(h, SZ), len(hidden), None)
    flat = np.zeros(P)
    ref.ref_artifact_init(S, A, seed, 1e-3, ptr(h, SZ), len(hidden), ptr(flat))
    return flat


def test_mlp_forward_and_log_prob_bit_exact(orc, ref):
    S, A = 13, 4
    flat = _flat_init(ref, S, A, 3, [16, 16])
    dims = _dims(S, 16, 16, A)
    pa = orc.orc_mlp_param_count(ptr(dims, SZ), 3)
    actor = np.ascontiguousarray(flat[:pa])
    X = np.random.default_rng(2).uniform(-2, 2, size=(9, S))
    y1 = np.zeros((9, A)); y2 = np.zeros((9, A))
    orc.orc_mlp_forward(ptr(actor), ptr(dims, SZ), 3, ptr(X), 9, ptr(y1), None)
    ref.ref_mlp_forward(ptr(actor), ptr(dims, SZ), 3, ptr(X), 9, ptr(y2))
    assert np.array_equal(y1, y2)
    ls = np.array([-0.3, 0.0, 0.2, -1.0])
    act = y1 + 0.37
    for i in range(9):
        assert orc.orc_gaussian_row_log_prob(ptr(ls), A, ptr(np.ascontiguousarray(y1[i])), ptr(np.ascontiguousarray(act[i]))) == \
            ref.ref_gaussian_row_log_prob(ptr(ls), A, ptr(np.ascontiguousarray(y1[i])), ptr(np.ascontiguousarray(act[i])))
    # nn.hpp test LogProbAtModePerDim (test_nn.cpp:249-257)
    lp = orc.orc_gaussian_row_log_prob(ptr(ls), A, ptr(np.ascontiguousarray(y1[0])), ptr(np.ascontiguousarray(y1[0])))
    assert abs(lp - sum(-0.5 * np.log(2 * np.pi) - ls)) < 1e-12


def test_gae_known_answers_and_reference(orc, ref):
    adv = np.zeros(1); ret = np.zeros(1)
    orc.orc_compute_gae(ptr(np.array([0.5])), ptr(np.array([2.0])), ptr(np.zeros(1, np.uint8), U8), 1, 3.0, 0.9,
                        0.95, ptr(adv), ptr(ret))  # test_ppo.cpp:71-75
    assert abs(adv[0] - (0.5 + 0.9 * 3.0 - 2.0)) < 1e-15 and abs(ret[0] - (adv[0] + 2.0)) < 1e-15
    rng = np.random.default_rng(3)
    for _ in range(20):
        T = int(rng.integers(1, 80))
        r = rng.uniform(-1, 1, T); v = rng.uniform(-1, 1, T); d = (rng.integers(0, 6, T) == 0).astype(np.uint8)
        b = float(rng.uniform(-1, 1))
        a1 = np.zeros(T); r1 = np.zeros(T); a2 = np.zeros(T); r2 = np.zeros(T)
        orc.orc_compute_gae(ptr(r), ptr(v), ptr(d, U8), T, b, 0.99, 0.95, ptr(a1), ptr(r1))
        ref.ref_compute_gae(ptr(r), ptr(v), ptr(d, U8), T, b, 0.99, 0.95, ptr(a2), ptr(r2))
        assert np.array_equal(a1, a2) and np.array_equal(r1, r2)


def test_buffer_advantages_normalised_bit_exact(orc, ref):
    rng = np.random.default_rng(4)
    N, H = 7, 33
    n = N * H
    r = rng.uniform(-1, 1, n); v = rng.uniform(-1, 1, n); d = (rng.integers(0, 9, n) == 0).astype(np.uint8)
    offs = np.arange(N, dtype=np.uint64) * H; lens = np.full(N, H, dtype=np.uint64); boot = rng.uniform(-1, 1, N)
    a1 = np.zeros(n); r1 = np.zeros(n); a2 = np.zeros(n); r2 = np.zeros(n)
    assert orc.orc_buffer_advantages(ptr(r), ptr(v), ptr(d, U8), n, ptr(offs, SZ), ptr(lens, SZ), ptr(boot), N,
                                     0.99, 0.95, 1, ptr(a1), ptr(r1)) == 0
    assert ref.ref_buffer_advantages(ptr(r), ptr(v), ptr(d, U8), n, ptr(offs, SZ), ptr(lens, SZ), ptr(boot), N,
                                     0.99, 0.95, 1, ptr(a2), ptr(r2)) == 0
    assert np.array_equal(a1, a2) and np.array_equal(r1, r2)
    # coverage check ppo.hpp:230-233
    assert orc.orc_buffer_advantages(ptr(r), ptr(v), ptr(d, U8), n, ptr(offs, SZ), ptr(lens, SZ), ptr(boot), N - 1,
                                     0.99, 0.95, 1, ptr(a1), ptr(r1)) == 3


def _cfg9(c: PpoCfg):
    return np.array([c.gamma, c.gae_lambda, c.clip_eps, c.entropy_coef, c.value_coef, c.epochs_per_update,
                     c.minibatch_size, c.buffer_size, c.learning_rate])


def test_ppo_loss_grads_bit_exact(orc, ref):
    S, A, hid = 11, 3, [8, 8]
    flat = _flat_init(ref, S, A, 5, hid)
    P = flat.size
    rng = np.random.default_rng(6)
    n = 37
    st = rng.uniform(-1, 1, (n, S)); ac = rng.uniform(-1, 1, (n, A)); olp = rng.uniform(-5, -2, n)
    adv = rng.normal(size=n); ret = rng.normal(size=n)
    cfg = PpoCfg(0.99, 0.95, 0.2, 0.01, 0.5, 4, n, n, 1e-3)
    g1 = np.zeros(P); g2 = np.zeros(P); l1 = np.zeros(3); l2 = np.zeros(3)
    ad = _dims(S, 8, 8, A); cd = _dims(S, 8, 8, 1)
    assert orc.orc_ppo_loss_grads(ptr(flat), ptr(ad, SZ), 3, ptr(cd, SZ), 3, ptr(st), ptr(ac), ptr(olp), ptr(adv),
                                  ptr(ret), n, C.byref(cfg), ptr(g1), ptr(l1)) == 0
    h = np.array(hid, dtype=np.uint64)
    assert ref.ref_ppo_loss_grads(ptr(flat), S, A, ptr(h, SZ), 2, ptr(st), ptr(ac), ptr(olp), ptr(adv), ptr(ret), n,
                                  ptr(_cfg9(cfg)), ptr(g2), ptr(l2)) == 0
    assert np.array_equal(l1, l2)
    assert np.array_equal(g1, g2)


def test_adam_known_answers_and_reference(orc, ref):
    # test_nn.cpp:199-208 FirstStepIsSignedLearningRate
    for g in (3.0, -0.7):
        p = np.zeros(1); m = np.zeros(1); v = np.zeros(1); t = C.c_int64(0)
        orc.orc_adam_step(ptr(p), ptr(np.array([g])), ptr(m), ptr(v), C.byref(t), 1, 0.9, 0.999, 1e-8, 1e-3)
        assert abs(p[0] + 1e-3 * np.sign(g)) < 1e-9
    # test_nn.cpp:228-234 non-finite grad aborts without touching state
    p = np.ones(1); m = np.zeros(1); v = np.zeros(1); t = C.c_int64(0)
    assert orc.orc_adam_step(ptr(p), ptr(np.array([np.nan])), ptr(m), ptr(v), C.byref(t), 1, 0.9, 0.999, 1e-8, 1e-3) == 2
    assert p[0] == 1.0 and t.value == 0
    rng = np.random.default_rng(8)
    P = 101
    p1 = rng.normal(size=P); m1 = np.zeros(P); v1 = np.zeros(P); t1 = C.c_int64(0)
    p2 = p1.copy(); m2 = m1.copy(); v2 = v1.copy(); t2 = C.c_int64(0)
    for _ in range(12):
        g = rng.normal(size=P)
        orc.orc_adam_step(ptr(p1), ptr(g), ptr(m1), ptr(v1), C.byref(t1), P, 0.9, 0.999, 1e-8, 1e-3)
        ref.ref_adam_step(ptr(p2), ptr(g), ptr(m2), ptr(v2), C.byref(t2), P, 1e-3)
    assert np.array_equal(p1, p2) and np.array_equal(m1, m2) and np.array_equal(v1, v2) and t1.value == t2.value


def test_ppo_update_with_reference_permutations_bit_exact(orc, ref):
    S, A, hid = 6, 2, [8, 8]
    flat = _flat_init(ref, S, A, 9, hid)
    P = flat.size
    N, H = 8, 16
    n = N * H
    rng = np.random.default_rng(10)
    st = rng.uniform(-1, 1, (n, S)); ac = rng.normal(size=(n, A)); lp = rng.uniform(-4, -1, n)
    rw = rng.normal(size=n); dn = (rng.integers(0, 10, n) == 0).astype(np.uint8); vl = rng.normal(size=n)
    offs = np.arange(N, dtype=np.uint64) * H; lens = np.full(N, H, dtype=np.uint64); boot = rng.normal(size=N)
    cfg = PpoCfg(0.99, 0.95, 0.2, 0.01, 0.5, 3, 32, n, 1e-3)
    seed = 1234
    perms = np.zeros(3 * n, dtype=np.uint64)
    ref.ref_ppo_permutations(seed, n, 3, ptr(perms, U64))
    f1 = flat.copy(); m1 = np.zeros(P); v1 = np.zeros(P); t1 = C.c_int64(0); s1 = np.zeros(4)
    ad = _dims(S, 8, 8, A); cd = _dims(S, 8, 8, 1)
    assert orc.orc_ppo_update(ptr(f1), ptr(m1), ptr(v1), C.byref(t1), ptr(ad, SZ), 3, ptr(cd, SZ), 3, ptr(st),
                              ptr(ac), ptr(lp), ptr(rw), ptr(dn, U8), ptr(vl), n, S, ptr(offs, SZ), ptr(lens, SZ),
                              ptr(boot), N, C.byref(cfg), ptr(perms, U64), ptr(s1)) == 0
    f2 = flat.copy(); m2 = np.zeros(P); v2 = np.zeros(P); t2 = C.c_int64(0); s2 = np.zeros(4)
    h = np.array(hid, dtype=np.uint64)
    assert ref.ref_ppo_update(ptr(f2), ptr(m2), ptr(v2), C.byref(t2), S, A, ptr(h, SZ), 2, ptr(st), ptr(ac), ptr(lp),
                              ptr(rw), ptr(dn, U8), ptr(vl), n, ptr(offs, SZ), ptr(lens, SZ), ptr(boot), N,
                              ptr(_cfg9(cfg)), seed, ptr(s2)) == 0
    assert t1.value == t2.value == 3 * (n // 32)
    assert np.array_equal(f1, f2) and np.array_equal(m1, m2) and np.array_equal(v1, v2)
    assert np.array_equal(s1, s2)


def test_fuse_bit_exact(orc, ref):
    S, A, hid = 5, 2, [4]
    P = _flat_init(ref, S, A, 1, hid).size
    rng = np.random.default_rng(12)
    L = 3
    ps = [rng.normal(size=P) for _ in range(L)]; ms = [rng.normal(size=P) for _ in range(L)]
    vs = [rng.uniform(0, 1, P) for _ in range(L)]; ts = np.array([5, 9, 7], dtype=np.int64)
    arr = lambda xs: (D * L)(*[ptr(x) for x in xs])
    o1 = [np.zeros(P) for _ in range(3)]; t1 = C.c_int64()
    orc.orc_fuse(arr(ps), arr(ms), arr(vs), ptr(ts, I64), L, P, ptr(o1[0]), ptr(o1[1]), ptr(o1[2]), C.byref(t1))
    o2 = [np.zeros(P) for _ in range(3)]; t2 = C.c_int64()
    h = np.array(hid, dtype=np.uint64)
    assert ref.ref_fuse(arr(ps), arr(ms), arr(vs), ptr(ts, I64), L, S, A, ptr(h, SZ), 1, ptr(o2[0]), ptr(o2[1]),
                        ptr(o2[2]), C.byref(t2)) == 0
    for a, b in zip(o1, o2):
        assert np.array_equal(a, b)
    assert t1.value == t2.value == 9


def test_leaderboard_matches_reference_with_ties(orc, ref):
    rng = np.random.default_rng(31)
    for trial in range(200):  # test_tournament.cpp:95-126 with forced ties
        cap = int(1 + rng.integers(0, 6)); n = int(1 + rng.integers(0, 30))
        scores = rng.uniform(-5, 5, n) if trial % 2 == 0 else rng.integers(0, 9, n).astype(np.float64)
        ids = np.arange(n, dtype=np.int64)
        bs = np.zeros(cap); bq = np.zeros(cap, dtype=np.uint64); bi = np.zeros(cap, dtype=np.int64)
        size = C.c_size_t(0); seq = C.c_uint64(0)
        ranks1 = [orc.orc_leaderboard_update(ptr(bs), ptr(bq, U64), ptr(bi, I64), C.byref(size), cap, C.byref(seq),
                                             float(s), int(i)) for s, i in zip(scores, ids)]
        oi = np.zeros(cap, dtype=np.int64); os_ = np.zeros(cap); osz = C.c_size_t(); rk = np.zeros(n, dtype=np.int64)
        assert ref.ref_leaderboard_sequence(ptr(scores), ptr(ids, I64), n, cap, ptr(oi, I64), ptr(os_),
                                            C.byref(osz), ptr(rk, I64)) == 0
        assert size.value == osz.value
        assert np.array_equal(bi[:size.value], oi[:osz.value])
        assert np.array_equal(np.array(ranks1), rk)


def test_population_stats_bit_exact(orc, ref):
    """Leaderboard::refresh_stats (tournament.hpp:66-87) after a leaderboard_update sequence of real
    64x64 stock artifacts: the oracle's mean / population variance over the final board's entries
    equals the reference's PopulationStats bit for bit."""
    from oracle_bind import population_stats
    rng = np.random.default_rng(5)
    S, A, hid = 181, 30, np.array([64, 64], dtype=np.uint64)
    P = 33661
    n, cap = 14, 10
    cand = rng.normal(scale=0.3, size=(n, P))
    scores = rng.integers(0, 6, n).astype(np.float64)
    ids = np.arange(n, dtype=np.int64)
    oi = np.full(cap, -1, np.int64); osz = C.c_size_t(); mean = np.zeros(P); var = np.zeros(P)
    assert ref.ref_leaderboard_stats(ptr(cand), ptr(scores), ptr(ids, I64), n, cap, S, A, ptr(hid, SZ), 2,
                                     ptr(oi, I64), C.byref(osz), ptr(mean), ptr(var)) == 0
    assert osz.value == cap
    om, ov = population_stats(orc, [cand[i] for i in oi[:osz.value]])
    assert np.array_equal(om, mean) and np.array_equal(ov, var)
