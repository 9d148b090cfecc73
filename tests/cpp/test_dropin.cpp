// test_dropin.cpp -- the C++ drop-in API (include/podracer_b200/podracer_b200.hpp)
// driven the way the reference's pod_train drives its own API (pod.hpp:353-485),
// checked against the C oracle (oracle/podracer_oracle.c, linked as test code).
// Run on a GPU box by tests/test_gpu_cpp.py; prints "DROPIN OK" on success.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <random>

#include "podracer_b200/podracer_b200.hpp"

extern "C" {
typedef struct {
  double initial_capital, max_trade_shares, cost_rate;
} orc_stock_cfg;
typedef struct {
  uint64_t mt[312];
  int idx;
} orc_mt64;
void orc_stock_vec_reset(size_t, int, const orc_stock_cfg*, size_t, double*, double*, size_t*, size_t*, double*);
int orc_stock_vec_step(size_t, int, const orc_stock_cfg*, size_t, size_t, const double*, const double*, size_t,
                       double*, double*, size_t*, size_t*, double*, const double*, double*, double*, uint8_t*, double*,
                       double*, uint64_t*);
void orc_pm_vec_reset(size_t, uint64_t, orc_mt64*, double*, uint64_t*, double*);
}

namespace pb = podracer_b200;

static int failures = 0;
#define EXPECT(cond)                                                   \
  do {                                                                 \
    if (!(cond)) {                                                     \
      std::fprintf(stderr, "FAILED %s:%d: %s\n", __FILE__, __LINE__, #cond); \
      ++failures;                                                      \
    }                                                                  \
  } while (0)

int main() {
  pb::Context ctx(0);
  const int K = 30;
  const size_t T = 160, N = 37, S = 1 + 6 * K;
  std::vector<double> open(K * T), high(K * T), low(K * T), close(K * T), vol(K * T), ind(4 * K * T);
  pb::check(prb_market_synthetic(2112, K, T, open.data(), high.data(), low.data(), close.data(), vol.data()));
  pb::check(prb_compute_indicators(high.data(), low.data(), close.data(), T, K, ind.data()));
  pb::MarketData market(ctx, close, &ind, T, K);
  pb::StockConfig cfg;
  cfg.initial_capital = 1e5;
  const size_t start = 10, end = 70;
  auto env = pb::VectorizedEnvironment::stock(market, cfg, start, end, N);
  EXPECT(env->spec().state_dim == S && env->spec().action_dim == (size_t)K);

  // ---- VecEnv parity against the oracle over two auto-resets ----
  orc_stock_cfg oc{cfg.initial_capital, cfg.max_trade_shares, cfg.cost_rate};
  std::vector<double> bal(N), sh(N * K), ret(N);
  std::vector<size_t> t(N), sc(N);
  orc_stock_vec_reset(N, K, &oc, start, bal.data(), sh.data(), t.data(), sc.data(), ret.data());
  pb::Tensor2 s0 = env->reset(3);
  EXPECT(s0.rows == N && s0.cols == S);
  std::mt19937_64 rng(9);
  std::uniform_real_distribution<double> u(-1.2, 1.2);
  size_t dones = 0;
  for (int step = 0; step < 130; ++step) {
    pb::Tensor2 a(N, K);
    for (auto& x : a.data) x = (double)(float)u(rng);  // the device consumes fp32 actions
    pb::VecStepResult r = env->step(a);
    std::vector<double> nx(N * S), rw(N), term(N * S), tr(N);
    std::vector<uint8_t> d(N);
    std::vector<uint64_t> tl(N);
    EXPECT(orc_stock_vec_step(N, K, &oc, start, end, close.data(), ind.data(), T, bal.data(), sh.data(), t.data(),
                              sc.data(), ret.data(), a.data.data(), nx.data(), rw.data(), d.data(), term.data(),
                              tr.data(), tl.data()) == 0);
    for (size_t i = 0; i < N; ++i) {
      EXPECT(r.dones[i] == d[i]);
      EXPECT((float)r.rewards[i] == (float)rw[i]);
      for (size_t j = 0; j < S; ++j) EXPECT((float)r.next_states.at(i, j) == (float)nx[i * S + j]);
      if (d[i]) {
        ++dones;
        EXPECT(r.infos[i].episode_end && r.infos[i].episode_length == tl[i] && r.infos[i].episode_return == tr[i]);
      }
    }
  }
  EXPECT(dones == 2 * N);
  bool threw = false;
  try {
    env->step(pb::Tensor2(N - 1, K));
  } catch (const pb::DimensionError&) {
    threw = true;
  }
  EXPECT(threw);

  // ---- PointMass resets are the reference's own per-env streams ----
  auto pm = pb::VectorizedEnvironment::pointmass(ctx, 16);
  pb::Tensor2 p0 = pm->reset(77);
  std::vector<orc_mt64> gens(16);
  std::vector<double> st(16 * 6), er(16);
  std::vector<uint64_t> psc(16);
  orc_pm_vec_reset(16, 77, gens.data(), st.data(), psc.data(), er.data());
  for (size_t i = 0; i < st.size(); ++i) EXPECT((float)p0.data[i] == (float)st[i]);

  // ---- one pod iteration: collect, GAE, PPO update, fusion of two learners ----
  auto actor = pb::Agent::init(ctx, S, K, 7, 1e-3);
  EXPECT(actor->param_count() == 33661);
  pb::PolicySample ps = pb::policy_sample(*actor, s0, 5);
  EXPECT(ps.actions.rows == N && ps.log_probs.size() == N);
  env->reset(4);
  const size_t H = 32;
  pb::TransitionBuffer buf(*env, H);
  pb::worker_collect(*actor, *env, buf, 11);
  auto [adv, ret2] = pb::buffer_advantages(buf, pb::PpoConfig{});
  double m = 0, v = 0;
  for (double x : adv) m += x;
  m /= adv.size();
  for (double x : adv) v += (x - m) * (x - m);
  v /= adv.size();
  EXPECT(std::fabs(m) < 1e-5 && std::fabs(v - 1.0) < 1e-3);
  pb::PpoConfig pc;
  pc.buffer_size = N * H;
  pc.minibatch_size = 128;
  pc.epochs_per_update = 2;
  auto l0 = pb::ppo_update(*actor, buf, pc, 1);
  auto l1 = pb::ppo_update(*actor, buf, pc, 2);
  EXPECT(l0.stats.minibatches == 2 * (N * H / 128));
  EXPECT(l0.artifact->optimizer_t() == (int64_t)l0.stats.minibatches);
  auto fused = pb::fuse_parameters({l0.artifact.get(), l1.artifact.get()});
  const auto f0 = l0.artifact->flatten_params(), f1 = l1.artifact->flatten_params(), ff = fused->flatten_params();
  for (size_t i = 0; i < ff.size(); ++i) EXPECT(std::fabs(ff[i] - 0.5 * (f0[i] + f1[i])) <= 1e-6 * (1 + std::fabs(ff[i])));
  const auto fa = actor->flatten_params();
  bool changed = false;
  for (size_t i = 0; i < fa.size(); ++i) changed |= fa[i] != f0[i];
  EXPECT(changed);  // trained copy differs; the input artifact is untouched (checked in the Python suite)
  threw = false;
  try {
    pb::PpoConfig bad = pc;
    bad.minibatch_size = pc.buffer_size * 2;
    pb::ppo_update(*actor, buf, bad, 1);
  } catch (const pb::ConfigError&) {
    threw = true;
  }
  EXPECT(threw);
  const std::vector<int> order = pb::leaderboard_rank(ctx, {1.0, 3.0, 3.0, 2.0}, {0, 1, 2, 3}, 3);
  EXPECT(order.size() == 3 && order[0] == 1 && order[1] == 2 && order[2] == 3);

  // generate_pod_init (tournament.hpp:136-162): the reference's draw order on the caller's rng,
  // the parent copied and mutated on the device, t := 0 with m / v kept, fresh path when empty
  {
    pb::GeneratorConfig gc;
    gc.top_k = 2;
    gc.fresh_prob = 0.3;
    gc.mutation_sigma = 0.05;
    auto fresh = [&](std::uint64_t seed) { return pb::Agent::init(ctx, S, K, seed, 1e-3); };
    std::vector<const pb::Agent*> board = {l0.artifact.get(), l1.artifact.get(), fused.get()};
    const std::vector<std::int64_t> ids = {11, 22, 33};
    int n_fresh = 0, n_child = 0;
    for (std::uint64_t seed = 1; seed <= 12; ++seed) {
      std::mt19937_64 rng(seed), replay(seed);
      pb::PodLineage lin;
      auto pod = pb::generate_pod_init(board, ids, gc, rng, fresh, &lin);
      // replay the reference's draws (tournament.hpp:142-153) on an identical generator
      std::uniform_real_distribution<double> u01(0.0, 1.0);
      if (u01(replay) < gc.fresh_prob) {
        const std::uint64_t fs = replay();
        EXPECT(lin.parent_pod == -1);
        EXPECT(pod->flatten_params() == pb::Agent::init(ctx, S, K, fs, 1e-3)->flatten_params());
        ++n_fresh;
      } else {
        std::uniform_int_distribution<std::size_t> pick(0, 1);
        const std::size_t i = pick(replay);
        const std::uint64_t ms = replay();
        EXPECT(lin.parent_pod == ids[i] && lin.mutation_seed == ms);
        EXPECT(pod->optimizer_t() == 0);
        const auto pp = board[i]->flatten_params(), cp = pod->flatten_params();
        double s1 = 0.0, s2 = 0.0;
        for (size_t j = 0; j < cp.size(); ++j) {
          const double dlt = cp[j] - pp[j];
          s1 += dlt;
          s2 += dlt * dlt;
        }
        const double mean = s1 / cp.size(), sd = std::sqrt(s2 / cp.size() - mean * mean);
        EXPECT(std::fabs(mean) < 5e-3 && std::fabs(sd - gc.mutation_sigma) < 5e-3);  // N(0, sigma^2) noise
        ++n_child;
      }
      EXPECT(rng() == replay());  // the caller's generator advanced exactly like the reference's
    }
    EXPECT(n_fresh > 0 && n_child > 0);
    std::mt19937_64 rng(5);
    pb::PodLineage lin;
    auto pod = pb::generate_pod_init({}, {}, gc, rng, fresh, &lin);  // empty board: fresh
    EXPECT(lin.parent_pod == -1 && pod->param_count() == l0.artifact->param_count());
  }

  // Leaderboard + leaderboard_update + refresh_stats (tournament.hpp:44-119): ties keep the earlier
  // arrival, a full board rejects scores <= its minimum, stats = mean / population variance of the
  // entries' params (on the device; checked here against a host restatement in the same order)
  {
    pb::Leaderboard lb(3);
    const double sc[] = {1.0, 3.0, 3.0, 0.5, 2.0, 3.0};
    std::vector<std::shared_ptr<const pb::Agent>> pods;
    int inserted = 0;
    for (int i = 0; i < 6; ++i) {
      pods.push_back(std::shared_ptr<const pb::Agent>(pb::Agent::init(ctx, S, K, 40 + i, 1e-3).release()));
      pb::LeaderboardEntry e;
      e.artifact = pods.back();
      e.score = sc[i];
      e.pod_id = i;
      inserted += pb::leaderboard_update(lb, e).inserted ? 1 : 0;
    }
    EXPECT(inserted == 5);  // 0.5 rejected once full (board {3,3,1} at that point)
    EXPECT(lb.size() == 3 && lb.at(0).pod_id == 1 && lb.at(1).pod_id == 2 && lb.at(2).pod_id == 5);
    const auto& st = lb.stats();
    std::vector<std::vector<double>> fl;
    for (const auto& e : lb.entries()) fl.push_back(e.artifact->flatten_params());
    bool same = st.mean.size() == fl[0].size();
    for (size_t j = 0; same && j < fl[0].size(); ++j) {
      double m = 0.0;
      for (const auto& f : fl) m += f[j];
      m *= 1.0 / 3.0;
      double v = 0.0;
      for (const auto& f : fl) v += (f[j] - m) * (f[j] - m);
      v *= 1.0 / 3.0;
      same = same && m == st.mean[j] && v == st.variance[j];
    }
    EXPECT(same);
    bool threw_nan = false;
    try {
      pb::LeaderboardEntry bad;
      bad.artifact = pods[0];
      bad.score = std::nan("");
      pb::leaderboard_update(lb, bad);
    } catch (const pb::NumericError&) {
      threw_nan = true;
    }
    EXPECT(threw_nan);
  }

  // ---- pods on one GPU: grouped collect, concurrent learners, device init, checkpoints ----
  {
    const size_t NP = 128, H = 32;
    std::vector<std::unique_ptr<pb::VectorizedEnvironment>> envs;
    std::vector<std::unique_ptr<pb::TransitionBuffer>> bufs, solo;
    std::vector<std::unique_ptr<pb::Agent>> agents;
    for (int p = 0; p < 2; ++p) {
      envs.push_back(pb::VectorizedEnvironment::stock(market, cfg, start, end, NP));
      envs.back()->reset(50 + p);
      bufs.push_back(std::make_unique<pb::TransitionBuffer>(*envs.back(), H));
      agents.push_back(pb::Agent::init(ctx, S, K, 60 + p, 1e-3));
    }
    pb::worker_collect_pods({agents[0].get(), agents[1].get()}, {envs[0].get(), envs[1].get()},
                            {bufs[0].get(), bufs[1].get()}, {70, 71});
    for (int p = 0; p < 2; ++p) {  // the same pods collected one by one
      auto e = pb::VectorizedEnvironment::stock(market, cfg, start, end, NP);
      e->reset(50 + p);
      solo.push_back(std::make_unique<pb::TransitionBuffer>(*e, H));
      pb::worker_collect(*agents[p], *e, *solo.back(), 70 + p);
      EXPECT(solo.back()->rewards() == bufs[p]->rewards());
    }
    pb::PpoConfig pc;
    pc.epochs_per_update = 1;
    pc.minibatch_size = 1024;
    pc.buffer_size = NP * H;
    for (auto& a : agents) a->set_ppo_mode(1);
    auto [outs, stats] = pb::ppo_update_learners({agents[0].get(), agents[1].get()}, {bufs[0].get(), bufs[1].get()},
                                                 pc, {80, 81});
    EXPECT(outs.size() == 2 && stats.size() == 2);
    for (int l = 0; l < 2; ++l) {  // each learner == its own ppo_update on the same path
      auto [one, st] = pb::ppo_update(*agents[l], *bufs[l], pc, 80 + l);
      EXPECT(one->flatten_params() == outs[l]->flatten_params());
      EXPECT(st.minibatches == stats[l].minibatches && st.mean_policy_loss == stats[l].mean_policy_loss);
      EXPECT(outs[l]->optimizer_t() == (int64_t)(NP * H / 1024));
    }
    {  // grouped evaluation == per-pod evaluation
      std::vector<std::unique_ptr<pb::VectorizedEnvironment>> ev;
      for (int p = 0; p < 2; ++p) ev.push_back(pb::VectorizedEnvironment::stock(market, cfg, start, end, 4));
      const auto recs = pb::evaluate_pods({outs[0].get(), outs[1].get()}, {ev[0].get(), ev[1].get()}, {5, 6});
      for (int p = 0; p < 2; ++p) {
        auto e1 = pb::VectorizedEnvironment::stock(market, cfg, start, end, 4);
        const pb::EvaluationRecord one = pb::evaluate(*outs[p], *e1, 5 + p);
        EXPECT(one.episodic_rewards == recs[p].episodic_rewards && one.mean == recs[p].mean);
      }
    }
    {  // the reference-signature overloads: worker_collect(..., rng) == worker_collect(..., rng())
      std::mt19937_64 r1(77), r2(77);
      auto e1 = pb::VectorizedEnvironment::stock(market, cfg, start, end, NP);
      auto e2 = pb::VectorizedEnvironment::stock(market, cfg, start, end, NP);
      e1->reset(3);
      e2->reset(3);
      pb::TransitionBuffer b1(*e1, H), b2(*e2, H);
      pb::worker_collect(*agents[0], *e1, H, b1, 0, 0, r1);
      pb::worker_collect(*agents[0], *e2, b2, r2());
      EXPECT(b1.rewards() == b2.rewards() && b1.actions() == b2.actions() && b1.states() == b2.states());
      EXPECT(b1.log_probs() == b2.log_probs() && b1.values() == b2.values() && b1.dones() == b2.dones());
      EXPECT(b1.states().size() == NP * H * S && b1.bootstrap_values().size() == NP && b1.full());
      bool threw_seg = false;
      try {
        pb::worker_collect(*agents[0], *e1, H, b1, 128, 0, r1);
      } catch (const pb::UsageError&) {
        threw_seg = true;
      }
      EXPECT(threw_seg);
      std::mt19937_64 r3(5), r4(5);
      pb::Tensor2 st(4, S);
      for (size_t i = 0; i < st.data.size(); ++i) st.data[i] = 0.01 * (double)(i % 97);
      const auto s1 = pb::policy_sample(*agents[0], st, r3);
      const auto s2 = pb::policy_sample(*agents[0], st, r4(), 0);
      EXPECT(s1.actions.data == s2.actions.data && s1.log_probs == s2.log_probs);
    }
    pb::Agent fresh(ctx, S, K);
    fresh.init_device(60, 1e-3);
    EXPECT(fresh.flatten_params() == agents[0]->flatten_params());
    const std::string path = "/tmp/podracer_b200_dropin.ckpt";
    pb::save_checkpoint(*outs[1], path, 4, 99);
    pb::Agent back(ctx, S, K);
    const pb::CheckpointInfo info = pb::load_checkpoint(back, path);
    EXPECT(info.parent_pod == 4 && info.mutation_seed == 99 && info.algo_tag == "ppo");
    EXPECT(back.flatten_params() == outs[1]->flatten_params() && back.optimizer_t() == outs[1]->optimizer_t());
    std::remove(path.c_str());
  }

  if (failures) {
    std::fprintf(stderr, "%d failures\n", failures);
    return 1;
  }
  std::printf("DROPIN OK\n");
  return 0;
}
