"""Generate tests/golden/ref_golden.npz from the REFERENCE ITSELF.

The vectors come from oracle/_ref/libpodracer_ref_exact.so, which is the
unmodified reference headers (/root/reference/cpp/include/podracer/*.hpp)
compiled behind a C shim by oracle/_ref's recipe.  This container has
/root/reference, so it can build that library.  A fresh clone or the GPU box
may not have it.  tests/test_golden.py checks the C restatement
(oracle/liboracle.so) against the committed file, so the oracle stays pinned
to the reference's outputs even where oracle/_ref cannot be built.

Run from the repo root after `python -c "import __graft_entry__ as g; g.build()"`:
    python tests/golden/make_golden.py
Reference calls used (all in the shim, following):
  derive_seed            common.hpp:79-105
  mt19937_64 / uniform   libstdc++ <random>, as env.hpp:124-133 draws them
  stock_env_step         stock_env.hpp:55-103
  indicators             stock_env.hpp / metrics (MACD, RSI, CCI, SMA)
  VectorizedEnvironment  env.hpp:167-249 (auto-reset, terminal infos)
  compute_gae            ppo.hpp:50-71
  buffer_advantages      ppo.hpp:212-244
  adam_step              nn.hpp:164-182
  leaderboard_update     tournament.hpp:44-119
"""
import ctypes as C
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
from oracle_bind import (MT64, derive_seed, indicators, load_ref, ptr, synthetic_market_np, I64,  # noqa: E402
                         SZ, U64, U8)


def main():
    ref = load_ref()
    if ref is None:
        raise SystemExit("oracle/_ref/libpodracer_ref_exact.so missing: build() in a container with /root/reference")
    out = {}
    rng = np.random.default_rng(2112)

    # derive_seed: 64 (base, tags...) cases, tags padded with -1 markers via a count column
    bases, tagm, cnt, seeds = [], [], [], []
    for _ in range(64):
        base = int(rng.integers(0, 2**63)); k = int(rng.integers(0, 4))
        tags = [int(x) for x in rng.integers(0, 2**40, size=k)]
        bases.append(base); cnt.append(k); tagm.append(tags + [0] * (3 - k))
        seeds.append(derive_seed(ref, base, *tags))
    out["ds_base"] = np.array(bases, np.uint64); out["ds_tags"] = np.array(tagm, np.uint64)
    out["ds_count"] = np.array(cnt, np.int64); out["ds_out"] = np.array(seeds, np.uint64)

    # mt19937_64 raw draws and uniform_real(-0.4, 0.4) (PointMass2D::reset)
    mt_seeds = np.array([0, 1, 5489, 2**63 + 7, 123456789], np.uint64)
    draws = np.zeros((len(mt_seeds), 700), np.uint64); unif = np.zeros((len(mt_seeds), 700))
    for i, s in enumerate(mt_seeds):
        ref.ref_mt64_draws(int(s), 700, ptr(draws[i], U64))
        ref.ref_uniform_real_draws(int(s), -0.4, 0.4, 700, ptr(unif[i]))
    out["mt_seeds"] = mt_seeds; out["mt_draws"] = draws; out["mt_unif"] = unif

    # single-env stock step sequences (sells then buys, affordability floor, costs)
    K, T = 5, 120
    close, high, low = synthetic_market_np(K, T, seed=3)
    out["st_close"] = close
    cfgs, acts, bals, shs, rews, dones = [], [], [], [], [], []
    for trial in range(6):
        cfg = (float(rng.choice([1e3, 1e5, 1e6])), float(rng.choice([10.0, 100.0])), float(rng.choice([0.0, 0.002])))
        a = rng.uniform(-1.5, 1.5, size=(T - 1, K))
        bal = C.c_double(cfg[0]); sh = np.zeros(K); t = C.c_size_t(0)
        tb, ts, tr, td = [], [], [], []
        for step in range(T - 1):
            r = C.c_double(); d = C.c_int()
            rc = ref.ref_stock_env_step(C.byref(bal), ptr(sh), C.byref(t), ptr(np.ascontiguousarray(a[step])),
                                        ptr(close), T, K, ptr(np.array(cfg)), C.byref(r), C.byref(d))
            assert rc == 0
            tb.append(bal.value); ts.append(sh.copy()); tr.append(r.value); td.append(d.value)
        cfgs.append(cfg); acts.append(a); bals.append(tb); shs.append(ts); rews.append(tr); dones.append(td)
    out["st_cfg"] = np.array(cfgs); out["st_actions"] = np.array(acts); out["st_balance"] = np.array(bals)
    out["st_shares"] = np.array(shs); out["st_reward"] = np.array(rews); out["st_done"] = np.array(dones, np.int32)

    # technical indicators
    c2, h2, l2 = synthetic_market_np(4, 300, seed=11)
    out["ind_close"] = c2; out["ind_high"] = h2; out["ind_low"] = l2; out["ind_out"] = indicators(ref, h2, l2, c2)

    # VecEnv with auto-reset (12-step episodes)
    K3, T3, N3 = 3, 80, 6
    c3, h3, l3 = synthetic_market_np(K3, T3, seed=5)
    ind3 = indicators(ref, h3, l3, c3)
    cfg3 = np.array([1e4, 100.0, 0.002]); start, end = 40, 52
    # fp32-representable actions: the device VecEnv takes its actions as fp32
    seq = np.array([rng.uniform(-1.2, 1.2, size=(N3, K3)).astype(np.float32).astype(np.float64) for _ in range(30)])
    S3 = 1 + 6 * K3
    h = ref.ref_stock_vec_create(ptr(c3), ptr(ind3), T3, K3, ptr(cfg3), start, end, N3)
    obs0 = np.zeros((N3, S3)); assert ref.ref_vec_reset(h, 9, ptr(obs0)) == 0
    vn, vr, vd, vt, vtr, vtl = [], [], [], [], [], []
    for acts_t in seq:
        e = [np.zeros((N3, S3)), np.zeros(N3), np.zeros(N3, np.uint8), np.zeros((N3, S3)), np.zeros(N3),
             np.zeros(N3, np.uint64)]
        assert ref.ref_vec_step(h, ptr(np.ascontiguousarray(acts_t)), K3, ptr(e[0]), ptr(e[1]), ptr(e[2], U8),
                                ptr(e[3]), ptr(e[4]), ptr(e[5], U64)) == 0
        m = e[2].astype(bool)
        e[3][~m] = 0; e[4][~m] = 0; e[5][~m] = 0  # infos exist only for done envs
        for lst, x in zip((vn, vr, vd, vt, vtr, vtl), e):
            lst.append(x)
    ref.ref_vec_destroy(h)
    out.update(vec_close=c3, vec_ind=ind3, vec_cfg=cfg3, vec_window=np.array([start, end]), vec_actions=seq,
               vec_obs0=obs0, vec_next=np.array(vn), vec_reward=np.array(vr), vec_done=np.array(vd),
               vec_term=np.array(vt), vec_term_ret=np.array(vtr), vec_term_len=np.array(vtl))

    # GAE over one chunk with dones, and buffer_advantages (normalised) over 7 chunks
    Tg = 77
    r = rng.uniform(-1, 1, Tg); v = rng.uniform(-1, 1, Tg); d = (rng.integers(0, 6, Tg) == 0).astype(np.uint8)
    b = float(rng.uniform(-1, 1)); ga = np.zeros(Tg); gr = np.zeros(Tg)
    ref.ref_compute_gae(ptr(r), ptr(v), ptr(d, U8), Tg, b, 0.99, 0.95, ptr(ga), ptr(gr))
    out.update(gae_r=r, gae_v=v, gae_d=d, gae_boot=np.array([b]), gae_adv=ga, gae_ret=gr)
    Nb, Hb = 7, 33; n = Nb * Hb
    r = rng.uniform(-1, 1, n); v = rng.uniform(-1, 1, n); d = (rng.integers(0, 9, n) == 0).astype(np.uint8)
    offs = np.arange(Nb, dtype=np.uint64) * Hb; lens = np.full(Nb, Hb, np.uint64); boot = rng.uniform(-1, 1, Nb)
    ba = np.zeros(n); br = np.zeros(n)
    assert ref.ref_buffer_advantages(ptr(r), ptr(v), ptr(d, U8), n, ptr(offs, SZ), ptr(lens, SZ), ptr(boot), Nb,
                                     0.99, 0.95, 1, ptr(ba), ptr(br)) == 0
    out.update(ba_r=r, ba_v=v, ba_d=d, ba_offs=offs, ba_lens=lens, ba_boot=boot, ba_adv=ba, ba_ret=br)

    # Adam: 12 steps over 101 params
    P = 101
    p = rng.normal(size=P); out["adam_p0"] = p.copy()
    m = np.zeros(P); vv = np.zeros(P); t = C.c_int64(0)
    gs = rng.normal(size=(12, P)); out["adam_g"] = gs
    for g in gs:
        ref.ref_adam_step(ptr(p), ptr(np.ascontiguousarray(g)), ptr(m), ptr(vv), C.byref(t), P, 1e-3)
    out.update(adam_p=p, adam_m=m, adam_v=vv, adam_t=np.array([t.value]))

    # leaderboard sequences with ties (capacity 1..6)
    lb_scores, lb_cap, lb_final, lb_ranks = [], [], [], []
    for trial in range(40):
        cap = int(1 + rng.integers(0, 6)); nn = 30
        s = rng.uniform(-5, 5, nn) if trial % 2 == 0 else rng.integers(0, 9, nn).astype(np.float64)
        ids = np.arange(nn, dtype=np.int64)
        oi = np.full(6, -1, np.int64); os_ = np.zeros(6); osz = C.c_size_t(); rk = np.zeros(nn, np.int64)
        assert ref.ref_leaderboard_sequence(ptr(s), ptr(ids, I64), nn, cap, ptr(oi, I64), ptr(os_), C.byref(osz),
                                            ptr(rk, I64)) == 0
        oi[osz.value:] = -1
        lb_scores.append(s); lb_cap.append(cap); lb_final.append(oi); lb_ranks.append(rk)
    out.update(lb_scores=np.array(lb_scores), lb_cap=np.array(lb_cap), lb_final=np.array(lb_final),
               lb_ranks=np.array(lb_ranks))

    path = os.path.join(HERE, "ref_golden.npz")
    np.savez_compressed(path, **out)
    print(f"wrote {path} ({os.path.getsize(path)} bytes, {len(out)} arrays)")


if __name__ == "__main__":
    main()
