"""Pin the C restatement (oracle/liboracle.so) against golden vectors that the
reference itself produced (tests/golden/ref_golden.npz, written by
tests/golden/make_golden.py through oracle/_ref, i.e. the unmodified reference
headers).  Unlike test_oracle_pinned.py this needs neither /root/reference nor
oracle/_ref, so the pin holds in a fresh clone and on the GPU box.  CPU only;
every comparison is bit-exact (np.array_equal)."""
import ctypes as C
import os

import numpy as np
import pytest

from oracle_bind import MT64, derive_seed, indicators, ptr, I64, SZ, U8
from test_oracle_pinned import _stock_step, _stock_vec_orc

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "ref_golden.npz")


@pytest.fixture(scope="module")
def g():
    return np.load(GOLDEN)


def test_derive_seed_golden(orc, g):  # common.hpp:79-105
    for base, tags, k, exp in zip(g["ds_base"], g["ds_tags"], g["ds_count"], g["ds_out"]):
        assert derive_seed(orc, int(base), *[int(x) for x in tags[:k]]) == int(exp)


def test_mt19937_64_and_uniform_golden(orc, g):  # env.hpp:124-133 draw order
    for i, s in enumerate(g["mt_seeds"]):
        st = MT64()
        orc.orc_mt64_seed(C.byref(st), int(s))
        got = np.array([orc.orc_mt64_next(C.byref(st)) for _ in range(700)], dtype=np.uint64)
        assert np.array_equal(got, g["mt_draws"][i])
        st = MT64()
        orc.orc_mt64_seed(C.byref(st), int(s))
        got = np.array([orc.orc_uniform_real(C.byref(st), -0.4, 0.4) for _ in range(700)])
        assert np.array_equal(got, g["mt_unif"][i])


def test_stock_step_sequences_golden(orc, g):  # stock_env.hpp:55-103
    close = np.ascontiguousarray(g["st_close"])
    K = close.shape[0]
    for trial in range(len(g["st_cfg"])):
        cfg = tuple(float(x) for x in g["st_cfg"][trial])
        bal, sh, t = cfg[0], np.zeros(K), 0
        for step, a in enumerate(g["st_actions"][trial]):
            rc, bal, sh, t, r, d = _stock_step(orc, "orc", bal, sh, t, a, close, cfg)
            assert rc == 0
            assert bal == g["st_balance"][trial][step]
            assert np.array_equal(sh, g["st_shares"][trial][step])
            assert r == g["st_reward"][trial][step] and d == g["st_done"][trial][step]


def test_indicators_golden(orc, g):
    got = indicators(orc, np.ascontiguousarray(g["ind_high"]), np.ascontiguousarray(g["ind_low"]),
                     np.ascontiguousarray(g["ind_close"]))
    assert np.array_equal(got, g["ind_out"])


def test_stock_vecenv_auto_reset_golden(orc, g):  # env.hpp:200-235
    start, end = (int(x) for x in g["vec_window"])
    cfg = tuple(float(x) for x in g["vec_cfg"])
    seq = [np.ascontiguousarray(a) for a in g["vec_actions"]]
    got = _stock_vec_orc(orc, np.ascontiguousarray(g["vec_close"]), np.ascontiguousarray(g["vec_ind"]), cfg, start,
                         end, seq[0].shape[0], seq)
    for s, (nxt, r, d, term, tr, tl) in enumerate(got):
        assert np.array_equal(nxt, g["vec_next"][s]) and np.array_equal(r, g["vec_reward"][s])
        assert np.array_equal(d, g["vec_done"][s])
        m = d.astype(bool)
        assert np.array_equal(term[m], g["vec_term"][s][m]) and np.array_equal(tr[m], g["vec_term_ret"][s][m])
        assert np.array_equal(tl[m], g["vec_term_len"][s][m])
    assert g["vec_done"].any()


def test_gae_and_buffer_advantages_golden(orc, g):  # ppo.hpp:50-71, 212-244
    r, v, d = (np.ascontiguousarray(g[k]) for k in ("gae_r", "gae_v", "gae_d"))
    T = r.size
    a = np.zeros(T); ret = np.zeros(T)
    orc.orc_compute_gae(ptr(r), ptr(v), ptr(d, U8), T, float(g["gae_boot"][0]), 0.99, 0.95, ptr(a), ptr(ret))
    assert np.array_equal(a, g["gae_adv"]) and np.array_equal(ret, g["gae_ret"])
    r, v, d, offs, lens, boot = (np.ascontiguousarray(g[k]) for k in
                                 ("ba_r", "ba_v", "ba_d", "ba_offs", "ba_lens", "ba_boot"))
    n = r.size
    a = np.zeros(n); ret = np.zeros(n)
    assert orc.orc_buffer_advantages(ptr(r), ptr(v), ptr(d, U8), n, ptr(offs, SZ), ptr(lens, SZ), ptr(boot),
                                     boot.size, 0.99, 0.95, 1, ptr(a), ptr(ret)) == 0
    assert np.array_equal(a, g["ba_adv"]) and np.array_equal(ret, g["ba_ret"])


def test_adam_golden(orc, g):  # nn.hpp:164-182
    p = g["adam_p0"].copy()
    P = p.size
    m = np.zeros(P); v = np.zeros(P); t = C.c_int64(0)
    for grad in g["adam_g"]:
        assert orc.orc_adam_step(ptr(p), ptr(np.ascontiguousarray(grad)), ptr(m), ptr(v), C.byref(t), P, 0.9, 0.999,
                                 1e-8, 1e-3) == 0
    assert np.array_equal(p, g["adam_p"]) and np.array_equal(m, g["adam_m"]) and np.array_equal(v, g["adam_v"])
    assert t.value == int(g["adam_t"][0])


def test_leaderboard_golden(orc, g):  # tournament.hpp:44-119, ranking indices bit-exact
    for scores, cap, final, ranks in zip(g["lb_scores"], g["lb_cap"], g["lb_final"], g["lb_ranks"]):
        cap = int(cap)
        bs = np.zeros(cap); bq = np.zeros(cap, dtype=np.uint64); bi = np.zeros(cap, dtype=np.int64)
        size = C.c_size_t(0); seq = C.c_uint64(0)
        got = [orc.orc_leaderboard_update(ptr(bs), ptr(bq, C.POINTER(C.c_uint64)), ptr(bi, I64), C.byref(size), cap,
                                          C.byref(seq), float(s), i) for i, s in enumerate(scores)]
        assert np.array_equal(np.array(got), ranks)
        assert np.array_equal(bi[:size.value], final[final >= 0])


GOLDEN_R2 = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "ref_golden_r2.npz")


@pytest.fixture(scope="module")
def g2():
    return np.load(GOLDEN_R2)


def test_population_stats_golden(orc, g2):  # Leaderboard::refresh_stats tournament.hpp:66-87
    from oracle_bind import population_stats
    for c, b, m, v in zip(g2["lbs_cand"], g2["lbs_board"], g2["lbs_mean"], g2["lbs_var"]):
        entries = [c[i].astype(np.float64) for i in b if i >= 0]
        om, ov = population_stats(orc, entries)
        assert np.array_equal(om, m) and np.array_equal(ov, v)
