// ref_shim.cpp -- TEST INFRASTRUCTURE ONLY.
//
// A thin extern "C" shim over the UNMODIFIED reference headers
// (/root/reference/proj/include/podracer/*.hpp, included read-only via -I).
// oracle/Makefile compiles it into oracle/_ref/ (git-ignored): one build with
// -ffp-contract=off (libpodracer_ref_exact.so, pins the C restatement
// bit-for-bit) and one with the reference's own release flags
// (libpodracer_ref_bench.so, the CPU baseline timed by bench.py --impl
// reference).  Nothing here is product code; every entry point just
// marshals plain arrays into the reference's own types and calls the
// reference function named in its comment.
#include <algorithm>
#include <chrono>
#include <cstdint>
#include <cstring>
#include <exception>
#include <memory>
#include <numeric>
#include <random>
#include <thread>
#include <vector>

#include "podracer/checkpoint.hpp"
#include "podracer/artifact.hpp"
#include "podracer/buffer.hpp"
#include "podracer/common.hpp"
#include "podracer/env.hpp"
#include "podracer/market.hpp"
#include "podracer/nn.hpp"
#include "podracer/pod.hpp"
#include "podracer/ppo.hpp"
#include "podracer/stock_env.hpp"
#include "podracer/tournament.hpp"

using namespace podracer;

#define REF_API extern "C" __attribute__((visibility("default")))

namespace {

int code_of(const std::exception& e) {
  if (dynamic_cast<const DimensionError*>(&e)) return 1;
  if (dynamic_cast<const NumericError*>(&e)) return 2;
  if (dynamic_cast<const UsageError*>(&e)) return 3;
  if (dynamic_cast<const FormatError*>(&e)) return 4;
  if (dynamic_cast<const DataError*>(&e)) return 5;
  if (dynamic_cast<const ConfigError*>(&e)) return 6;
  if (dynamic_cast<const CorruptionError*>(&e)) return 7;
  if (dynamic_cast<const VersionError*>(&e)) return 8;
  if (dynamic_cast<const DomainError*>(&e)) return 9;
  return 99;
}

#define GUARD(...)                           \
  try {                                      \
    __VA_ARGS__;                             \
    return 0;                                \
  } catch (const std::exception& e) {        \
    return code_of(e);                       \
  }

// close[k*T+t], indicators[(i*K+k)*T+t]
std::shared_ptr<MarketData> make_market(const double* close, const double* indicators, size_t T, int K) {
  auto d = std::make_shared<MarketData>();
  for (int k = 0; k < K; ++k) d->tickers.push_back("T" + std::to_string(k));
  d->series.resize(K);
  for (size_t t = 0; t < T; ++t) d->timestamps.push_back(static_cast<std::int64_t>(t) * 60);
  for (int k = 0; k < K; ++k) {
    auto& s = d->series[k];
    s.close.assign(close + (size_t)k * T, close + (size_t)(k + 1) * T);
    s.open = s.close;
    s.high = s.close;
    s.low = s.close;
    s.volume.assign(T, 1000.0);
    if (indicators) {
      s.indicators.resize(4);
      for (int i = 0; i < 4; ++i) {
        const double* p = indicators + ((size_t)i * K + k) * T;
        s.indicators[i].assign(p, p + T);
      }
    }
  }
  return d;
}

std::vector<std::size_t> dims_of(const size_t* d, int n) { return std::vector<std::size_t>(d, d + n); }

struct RefAgentShape {
  std::size_t S, A;
  std::vector<std::size_t> hidden;
};

AgentArtifact artifact_from(const double* flat, const double* m, const double* v, int64_t t, size_t S, size_t A,
                            const size_t* hidden, int nh, double lr) {
  AgentArtifact a = artifact_init(S, A, 0, lr, dims_of(hidden, nh));
  std::vector<double> f(flat, flat + a.param_count());
  a.unflatten_params(f);
  if (m) a.optimizer.m.assign(m, m + a.param_count());
  if (v) a.optimizer.v.assign(v, v + a.param_count());
  a.optimizer.t = t;
  return a;
}

}  // namespace

REF_API uint64_t ref_derive_seed(uint64_t base, const uint64_t* tags, int ntags) {
  switch (ntags) {
    case 0: return derive_seed(base);
    case 1: return derive_seed(base, tags[0]);
    case 2: return derive_seed(base, tags[0], tags[1]);
    case 3: return derive_seed(base, tags[0], tags[1], tags[2]);
    default: return 0;
  }
}

// std::mt19937_64 + uniform_real_distribution draws (env.hpp:124-133 uses them).
REF_API void ref_uniform_real_draws(uint64_t seed, double a, double b, size_t n, double* out) {
  std::mt19937_64 rng(seed);
  std::uniform_real_distribution<double> u(a, b);
  for (size_t i = 0; i < n; ++i) out[i] = u(rng);
}

REF_API void ref_mt64_draws(uint64_t seed, size_t n, uint64_t* out) {
  std::mt19937_64 rng(seed);
  for (size_t i = 0; i < n; ++i) out[i] = rng();
}

// ---- stock env: stock_env_step stock_env.hpp:55 ---------------------------
REF_API int ref_stock_env_step(double* balance, double* shares, size_t* t, const double* action, const double* close,
                               size_t T, int K, const double* cfg3, double* reward, int* done) {
  GUARD({
    auto data = make_market(close, nullptr, T, K);
    StockConfig cfg{cfg3[0], cfg3[1], cfg3[2]};
    PortfolioState s;
    s.balance = *balance;
    s.shares.assign(shares, shares + K);
    s.t = *t;
    std::vector<double> a(action, action + K);
    StockStep r = stock_env_step(s, a, *data, cfg);
    *balance = r.state.balance;
    std::copy(r.state.shares.begin(), r.state.shares.end(), shares);
    *t = r.state.t;
    *reward = r.reward;
    *done = r.done ? 1 : 0;
  })
}

// ---- VecEnv over StockTradingEnv / PointMass2D: env.hpp:167-249 ----------
struct RefVec {
  std::shared_ptr<MarketData> data;
  std::unique_ptr<VectorizedEnvironment> venv;
};

REF_API void* ref_stock_vec_create(const double* close, const double* indicators, size_t T, int K, const double* cfg3,
                                   size_t start, size_t end, size_t N) {
  auto* h = new RefVec;
  h->data = make_market(close, indicators, T, K);
  StockConfig cfg{cfg3[0], cfg3[1], cfg3[2]};
  auto data = h->data;
  h->venv = std::make_unique<VectorizedEnvironment>(
      [data, cfg, start, end] { return std::make_unique<StockTradingEnv>(data, cfg, start, end); }, N);
  return h;
}

REF_API void* ref_pm_vec_create(size_t N) {
  auto* h = new RefVec;
  h->venv = std::make_unique<VectorizedEnvironment>([] { return std::make_unique<PointMass2D>(); }, N);
  return h;
}

REF_API void ref_vec_destroy(void* h) { delete static_cast<RefVec*>(h); }

REF_API int ref_vec_reset(void* hh, uint64_t seed, double* obs) {
  GUARD({
    auto* h = static_cast<RefVec*>(hh);
    Tensor2 s = h->venv->reset(seed);
    std::copy(s.data.begin(), s.data.end(), obs);
  })
}

REF_API int ref_vec_step(void* hh, const double* actions, size_t A, double* next_obs, double* reward, uint8_t* done,
                         double* terminal_obs, double* term_return, uint64_t* term_len) {
  GUARD({
    auto* h = static_cast<RefVec*>(hh);
    const size_t N = h->venv->num_envs();
    Tensor2 act(N, A);
    std::copy(actions, actions + N * A, act.data.begin());
    VecStepResult r = h->venv->step(act);
    const size_t S = r.next_states.cols;
    std::copy(r.next_states.data.begin(), r.next_states.data.end(), next_obs);
    for (size_t e = 0; e < N; ++e) {
      reward[e] = r.rewards[e];
      done[e] = r.dones[e];
      if (r.infos[e].episode_end) {
        std::copy(r.infos[e].terminal_state.begin(), r.infos[e].terminal_state.end(), terminal_obs + e * S);
        term_return[e] = r.infos[e].episode_return;
        term_len[e] = r.infos[e].episode_length;
      }
    }
  })
}

REF_API void ref_vec_step_counts(void* hh, uint64_t* out) {
  auto* h = static_cast<RefVec*>(hh);
  const auto& c = h->venv->step_counts();
  for (size_t i = 0; i < c.size(); ++i) out[i] = c[i];
}

REF_API int ref_pointmass_step(const double* s, const double* a, uint64_t steps, double* out, double* reward,
                               int* done) {
  GUARD({
    PointMassStep r = pointmass_step(std::vector<double>(s, s + 6), std::vector<double>(a, a + 2), steps);
    std::copy(r.next_state.begin(), r.next_state.end(), out);
    *reward = r.reward;
    *done = r.done ? 1 : 0;
  })
}

// ---- market: compute_indicators market.hpp:373 ----------------------------
REF_API int ref_compute_indicators(const double* high, const double* low, const double* close, size_t T, int K,
                                   double* out) {
  GUARD({
    auto d = make_market(close, nullptr, T, K);
    for (int k = 0; k < K; ++k) {
      d->series[k].high.assign(high + (size_t)k * T, high + (size_t)(k + 1) * T);
      d->series[k].low.assign(low + (size_t)k * T, low + (size_t)(k + 1) * T);
    }
    MarketData m = compute_indicators(*d);
    for (int k = 0; k < K; ++k)
      for (int i = 0; i < 4; ++i)
        std::copy(m.series[k].indicators[i].begin(), m.series[k].indicators[i].end(), out + ((size_t)i * K + k) * T);
  })
}

// ---- NN: mlp_forward nn.hpp:63, gaussian_log_prob :229, adam_step :164 -----
REF_API int ref_mlp_forward(const double* params, const size_t* dims, int nlayers, const double* X, size_t n,
                            double* Y) {
  GUARD({
    MlpParams p = mlp_init(dims_of(dims, nlayers + 1), 0);
    const double* q = params;
    for (auto& l : p.layers) {
      std::copy(q, q + l.weight.size(), l.weight.data.begin());
      q += l.weight.size();
      std::copy(q, q + l.bias.size(), l.bias.begin());
      q += l.bias.size();
    }
    Tensor2 in(n, dims[0]);
    std::copy(X, X + n * dims[0], in.data.begin());
    Tensor2 out = mlp_forward(p, in);
    std::copy(out.data.begin(), out.data.end(), Y);
  })
}

REF_API double ref_gaussian_row_log_prob(const double* log_std, int A, const double* mean, const double* action) {
  std::vector<double> ls(log_std, log_std + A);
  return detail::gaussian_row_log_prob(ls, mean, action);
}

REF_API int ref_adam_step(double* params, const double* grads, double* m, double* v, int64_t* t, size_t n, double lr) {
  GUARD({
    std::vector<double> p(params, params + n), g(grads, grads + n);
    AdamState s = adam_init(n, lr);
    s.m.assign(m, m + n);
    s.v.assign(v, v + n);
    s.t = *t;
    adam_step(p, g, s);
    std::copy(p.begin(), p.end(), params);
    std::copy(s.m.begin(), s.m.end(), m);
    std::copy(s.v.begin(), s.v.end(), v);
    *t = s.t;
  })
}

// ---- artifact_init artifact.hpp:91 (canonical flat layout) -----------------
REF_API size_t ref_artifact_init(size_t S, size_t A, uint64_t seed, double lr, const size_t* hidden, int nh,
                                 double* flat_out) {
  AgentArtifact a = artifact_init(S, A, seed, lr, dims_of(hidden, nh));
  std::vector<double> f = a.flatten_params();
  if (flat_out) std::copy(f.begin(), f.end(), flat_out);
  return f.size();
}

// ---- GAE: compute_gae ppo.hpp:50, buffer_advantages :212 -------------------
REF_API int ref_compute_gae(const double* r, const double* v, const uint8_t* d, size_t T, double bootstrap,
                            double gamma, double lambda, double* adv, double* ret) {
  GUARD({
    GaeResult g = compute_gae(std::vector<double>(r, r + T), std::vector<double>(v, v + T),
                              std::vector<std::uint8_t>(d, d + T), bootstrap, gamma, lambda);
    std::copy(g.advantages.begin(), g.advantages.end(), adv);
    std::copy(g.returns.begin(), g.returns.end(), ret);
  })
}

static TransitionBuffer make_buffer(const double* states, const double* actions, const double* log_probs,
                                    const double* rewards, const uint8_t* dones, const double* values, size_t n,
                                    size_t S, size_t A, const size_t* offsets, const size_t* lengths,
                                    const double* bootstrap, size_t nchunks) {
  TransitionBuffer buf(n, S, A);
  buf.commit_segment(0, n);
  Transition tr;
  tr.state.resize(S);
  tr.action.resize(A);
  for (size_t i = 0; i < n; ++i) {
    if (states) std::copy(states + i * S, states + (i + 1) * S, tr.state.begin());
    if (actions) std::copy(actions + i * A, actions + (i + 1) * A, tr.action.begin());
    tr.log_prob = log_probs ? log_probs[i] : 0.0;
    tr.reward = rewards[i];
    tr.done = dones[i] != 0;
    tr.value = values[i];
    buf.put(i, tr);
  }
  for (size_t c = 0; c < nchunks; ++c) buf.add_chunk(offsets[c], lengths[c], bootstrap[c]);
  return buf;
}

REF_API int ref_buffer_advantages(const double* r, const double* v, const uint8_t* d, size_t n, const size_t* offsets,
                                  const size_t* lengths, const double* bootstrap, size_t nchunks, double gamma,
                                  double lambda, int normalize, double* adv, double* ret) {
  GUARD({
    TransitionBuffer buf = make_buffer(nullptr, nullptr, nullptr, r, d, v, n, 1, 1, offsets, lengths, bootstrap, nchunks);
    PpoConfig cfg;
    cfg.gamma = gamma;
    cfg.gae_lambda = lambda;
    GaeResult g = buffer_advantages(buf, cfg, normalize != 0);
    std::copy(g.advantages.begin(), g.advantages.end(), adv);
    std::copy(g.returns.begin(), g.returns.end(), ret);
  })
}

static PpoConfig ppo_cfg_from(const double* c) {
  // c = gamma, lambda, clip, ent, vf, epochs, minibatch, buffer, lr
  PpoConfig cfg;
  cfg.gamma = c[0];
  cfg.gae_lambda = c[1];
  cfg.clip_eps = c[2];
  cfg.entropy_coef = c[3];
  cfg.value_coef = c[4];
  cfg.epochs_per_update = static_cast<std::size_t>(c[5]);
  cfg.minibatch_size = static_cast<std::size_t>(c[6]);
  cfg.buffer_size = static_cast<std::size_t>(c[7]);
  cfg.learning_rate = c[8];
  return cfg;
}

// detail::ppo_loss_grads ppo.hpp:116 on an explicit minibatch.
REF_API int ref_ppo_loss_grads(const double* flat, size_t S, size_t A, const size_t* hidden, int nh,
                               const double* mb_states, const double* mb_actions, const double* mb_old_lp,
                               const double* mb_adv, const double* mb_ret, size_t n, const double* cfg9,
                               double* grads, double* losses) {
  GUARD({
    AgentArtifact a = artifact_from(flat, nullptr, nullptr, 0, S, A, hidden, nh, 1e-3);
    Minibatch mb;
    mb.states = Tensor2(n, S);
    std::copy(mb_states, mb_states + n * S, mb.states.data.begin());
    mb.actions = Tensor2(n, A);
    std::copy(mb_actions, mb_actions + n * A, mb.actions.data.begin());
    mb.old_log_probs.assign(mb_old_lp, mb_old_lp + n);
    mb.advantages.assign(mb_adv, mb_adv + n);
    mb.returns.assign(mb_ret, mb_ret + n);
    std::vector<double> g;
    PpoLosses l = detail::ppo_loss_grads(a.actor, a.critic, mb, ppo_cfg_from(cfg9), grads ? &g : nullptr);
    if (grads) std::copy(g.begin(), g.end(), grads);
    losses[0] = l.policy_loss;
    losses[1] = l.value_loss;
    losses[2] = l.entropy;
  })
}

// The permutation sequence ppo_update ppo.hpp:271-274 draws for `seed`.
REF_API void ref_ppo_permutations(uint64_t seed, size_t n, size_t epochs, uint64_t* out) {
  std::mt19937_64 rng(seed);
  std::vector<std::size_t> idx(n);
  std::iota(idx.begin(), idx.end(), 0);
  for (size_t e = 0; e < epochs; ++e) {
    std::shuffle(idx.begin(), idx.end(), rng);
    for (size_t j = 0; j < n; ++j) out[e * n + j] = idx[j];
  }
}

// ppo_update ppo.hpp:249 (the real one, std::shuffle inside).
REF_API int ref_ppo_update(double* flat, double* m, double* v, int64_t* t, size_t S, size_t A, const size_t* hidden,
                           int nh, const double* states, const double* actions, const double* log_probs,
                           const double* rewards, const uint8_t* dones, const double* values, size_t n,
                           const size_t* offsets, const size_t* lengths, const double* bootstrap, size_t nchunks,
                           const double* cfg9, uint64_t seed, double* stats) {
  GUARD({
    PpoConfig cfg = ppo_cfg_from(cfg9);
    AgentArtifact a = artifact_from(flat, m, v, *t, S, A, hidden, nh, cfg.learning_rate);
    TransitionBuffer buf =
        make_buffer(states, actions, log_probs, rewards, dones, values, n, S, A, offsets, lengths, bootstrap, nchunks);
    PpoUpdateResult r = ppo_update(a, buf, cfg, seed);
    std::vector<double> f = r.artifact.flatten_params();
    std::copy(f.begin(), f.end(), flat);
    std::copy(r.artifact.optimizer.m.begin(), r.artifact.optimizer.m.end(), m);
    std::copy(r.artifact.optimizer.v.begin(), r.artifact.optimizer.v.end(), v);
    *t = r.artifact.optimizer.t;
    stats[0] = r.stats.mean_policy_loss;
    stats[1] = r.stats.mean_value_loss;
    stats[2] = r.stats.mean_entropy;
    stats[3] = static_cast<double>(r.stats.minibatches);
  })
}

// ---- fuse_parameters pod.hpp:141 -------------------------------------------
REF_API int ref_fuse(const double* const* params, const double* const* m, const double* const* v, const int64_t* t,
                     size_t L, size_t S, size_t A, const size_t* hidden, int nh, double* out_p, double* out_m,
                     double* out_v, int64_t* out_t) {
  GUARD({
    std::vector<AgentArtifact> arts;
    for (size_t i = 0; i < L; ++i) arts.push_back(artifact_from(params[i], m[i], v[i], t[i], S, A, hidden, nh, 1e-3));
    AgentArtifact f = fuse_parameters(arts);
    std::vector<double> fp = f.flatten_params();
    std::copy(fp.begin(), fp.end(), out_p);
    std::copy(f.optimizer.m.begin(), f.optimizer.m.end(), out_m);
    std::copy(f.optimizer.v.begin(), f.optimizer.v.end(), out_v);
    *out_t = f.optimizer.t;
  })
}

// ---- leaderboard_update tournament.hpp:104 over a candidate sequence -------
// Inserts scores[i] (pod ids[i]) in order; writes the final board's pod ids
// (rank order) to out_ids and each call's returned rank (-1 = rejected) to ranks.
REF_API int ref_leaderboard_sequence(const double* scores, const int64_t* ids, size_t n, size_t capacity,
                                     int64_t* out_ids, double* out_scores, size_t* out_size, int64_t* ranks) {
  GUARD({
    Leaderboard board(capacity);
    AgentArtifact tiny = artifact_init(1, 1, 0, 1e-3, {1});
    for (size_t i = 0; i < n; ++i) {
      LeaderboardEntry e;
      e.artifact = tiny;
      e.score = scores[i];
      e.pod_id = ids[i];
      LeaderboardUpdate u = leaderboard_update(board, e);
      ranks[i] = u.inserted ? static_cast<int64_t>(*u.rank) : -1;
    }
    *out_size = board.size();
    for (size_t r = 0; r < board.size(); ++r) {
      out_ids[r] = board.at(r).pod_id;
      out_scores[r] = board.at(r).score;
    }
  })
}

// ---- leaderboard_update + refresh_stats tournament.hpp:66-119 with real artifacts ----
// Candidate i carries flat params cand[i*P .. i*P+P) of an S-hidden-A agent.  Inserts them in
// order; writes the final board's pod ids (rank order) and the board's PopulationStats.
REF_API int ref_leaderboard_stats(const double* cand, const double* scores, const int64_t* ids, size_t n,
                                  size_t capacity, size_t S, size_t A, const size_t* hidden, int nh,
                                  int64_t* out_ids, size_t* out_size, double* mean, double* variance) {
  GUARD({
    Leaderboard board(capacity);
    size_t P = 0;
    for (size_t i = 0; i < n; ++i) {
      LeaderboardEntry e;
      e.artifact = artifact_init(S, A, 0, 1e-3, dims_of(hidden, nh));
      P = e.artifact.param_count();
      e.artifact.unflatten_params(std::vector<double>(cand + i * P, cand + (i + 1) * P));
      e.score = scores[i];
      e.pod_id = ids[i];
      leaderboard_update(board, e);
    }
    *out_size = board.size();
    for (size_t r = 0; r < board.size(); ++r) out_ids[r] = board.at(r).pod_id;
    const PopulationStats& st = board.stats();
    std::copy(st.mean.begin(), st.mean.end(), mean);
    std::copy(st.variance.begin(), st.variance.end(), variance);
  })
}

// ---- checkpoints (checkpoint.hpp): an artifact from flat params / Adam state -> the reference's
// own encode_checkpoint(artifact_to_tensors(...)) bytes, and decode + artifact_from_tensors back.
// Returns the byte count (out may be NULL to size), or (size_t)-1 on error.
REF_API size_t ref_checkpoint_encode(const double* flat, const double* m, const double* v, int64_t t,
                                     const double* hyper, size_t S, size_t A, const size_t* hidden, int nh,
                                     int64_t parent, uint64_t mseed, const char* tag, const double* meta,
                                     uint8_t* out) {
  try {
    AgentArtifact a = artifact_from(flat, m, v, t, S, A, hidden, nh, hyper[3]);
    a.optimizer.beta1 = hyper[0];
    a.optimizer.beta2 = hyper[1];
    a.optimizer.eps = hyper[2];
    a.lineage.parent_pod = parent;
    a.lineage.mutation_seed = mseed;
    a.algo_tag = tag;
    CheckpointMeta cm;
    if (meta) {
      cm.wall_seconds = meta[0];
      cm.env_steps = meta[1];
      cm.score = meta[2];
    }
    const std::vector<std::uint8_t> b = encode_checkpoint(artifact_to_tensors(a, meta ? &cm : nullptr));
    if (out) std::copy(b.begin(), b.end(), out);
    return b.size();
  } catch (...) {
    return (size_t)-1;
  }
}

// decode_checkpoint + artifact_from_tensors; returns 0, or the error class: 7 corruption, 4 format,
// 8 version, 99 other.  flat/m/v sized by the caller (the artifact's param_count).
REF_API int ref_checkpoint_decode(const uint8_t* bytes, size_t n, double* flat, double* m, double* v, int64_t* t,
                                  int64_t* parent, uint64_t* mseed) {
  try {
    AgentArtifact a = artifact_from_tensors(decode_checkpoint(std::vector<std::uint8_t>(bytes, bytes + n)));
    const std::vector<double> f = a.flatten_params();
    std::copy(f.begin(), f.end(), flat);
    std::copy(a.optimizer.m.begin(), a.optimizer.m.end(), m);
    std::copy(a.optimizer.v.begin(), a.optimizer.v.end(), v);
    *t = a.optimizer.t;
    *parent = a.lineage.parent_pod;
    *mseed = a.lineage.mutation_seed;
    return 0;
  } catch (const CorruptionError&) {
    return 7;
  } catch (const FormatError&) {
    return 4;
  } catch (const VersionError&) {
    return 8;
  } catch (...) {
    return 99;
  }
}

// ppo_update ppo.hpp:249 timing on a synthetic buffer of n transitions (chunks of
// `horizon`; states/actions/log-probs/values/rewards from mt19937_64(seed)),
// `epochs` x (n / minibatch) sequential Adam steps.  Returns wall seconds.
REF_API double ref_bench_ppo(const double* flat, size_t S, size_t A, const size_t* hidden, int nh, size_t n,
                             size_t horizon, size_t minibatch, size_t epochs, uint64_t seed) {
  std::mt19937_64 rng(seed);
  std::normal_distribution<double> nd(0.0, 1.0);
  std::vector<double> st(n * S), ac(n * A), lp(n), rw(n), vl(n);
  std::vector<uint8_t> dn(n, 0);
  for (auto& x : st) x = nd(rng);
  for (auto& x : ac) x = nd(rng);
  for (size_t i = 0; i < n; ++i) {
    lp[i] = -0.5 * (double)A + 0.1 * nd(rng);
    rw[i] = nd(rng);
    vl[i] = nd(rng);
  }
  const size_t nch = n / horizon;
  std::vector<size_t> off(nch), len(nch, horizon);
  std::vector<double> boot(nch, 0.0);
  for (size_t c = 0; c < nch; ++c) off[c] = c * horizon;
  TransitionBuffer buf = make_buffer(st.data(), ac.data(), lp.data(), rw.data(), dn.data(), vl.data(), n, S, A,
                                     off.data(), len.data(), boot.data(), nch);
  AgentArtifact a = artifact_from(flat, nullptr, nullptr, 0, S, A, hidden, nh, 1e-3);
  PpoConfig cfg;
  cfg.epochs_per_update = epochs;
  cfg.minibatch_size = minibatch;
  cfg.buffer_size = n;
  auto t0 = std::chrono::steady_clock::now();
  PpoUpdateResult r = ppo_update(a, buf, cfg, seed);
  const double s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  return r.stats.minibatches > 0 ? s : -1.0;
}

// ---- CPU baseline timing (bench.py --impl reference / cpu_baseline) --------
// The bench's synthetic market (the reference ships no generator): mt19937_64(seed);
// p0_k ~ U(10,200) for k = 0..K-1, then for t = 1..T-1, k = 0..K-1: p_k[t] = p_k[t-1] * exp(1e-3 N(0,1));
// high = 1.001 p, low = 0.999 p.  Arrays [K][T].  Lets the reference arm build its inputs without
// the product library.
REF_API void ref_synthetic_market(uint64_t seed, int K, size_t T, double* close, double* high, double* low) {
  std::mt19937_64 rng(seed);
  std::uniform_real_distribution<double> u0(10.0, 200.0);
  std::normal_distribution<double> nrm(0.0, 1.0);
  for (int k = 0; k < K; ++k) close[(size_t)k * T] = u0(rng);
  for (size_t t = 1; t < T; ++t)
    for (int k = 0; k < K; ++k) close[(size_t)k * T + t] = close[(size_t)k * T + t - 1] * std::exp(1e-3 * nrm(rng));
  for (size_t i = 0; i < (size_t)K * T; ++i) {
    high[i] = 1.001 * close[i];
    low[i] = 0.999 * close[i];
  }
}

// pod_train's collect phase (pod.hpp:408-433): `workers` threads, each owning
// a VectorizedEnvironment of envs_per_worker stock envs, running worker_collect
// for `horizon` steps into disjoint segments of one shared buffer.
// Returns wall seconds; transitions = workers*envs_per_worker*horizon.
REF_API double ref_bench_collect(const double* close, const double* indicators, size_t T, int K, size_t start,
                                 size_t end, size_t workers, size_t envs_per_worker, size_t horizon,
                                 const double* flat, const size_t* hidden, int nh, uint64_t seed) {
  auto data = make_market(close, indicators, T, K);
  StockConfig cfg;
  const size_t S = stock_observation_dim(K);
  AgentArtifact art = artifact_from(flat, nullptr, nullptr, 0, S, K, hidden, nh, 1e-3);
  EnvFactory factory = [data, cfg, start, end] { return std::make_unique<StockTradingEnv>(data, cfg, start, end); };
  std::vector<std::unique_ptr<VectorizedEnvironment>> venvs;
  for (size_t w = 0; w < workers; ++w) {
    venvs.push_back(std::make_unique<VectorizedEnvironment>(factory, envs_per_worker));
    venvs[w]->reset(derive_seed(seed, seed_tag::kVecEnv, w));
  }
  const size_t seg = envs_per_worker * horizon;
  TransitionBuffer buffer(workers * seg, S, K);
  auto t0 = std::chrono::steady_clock::now();
  buffer.clear();
  buffer.resize_chunks(workers * envs_per_worker);
  for (size_t w = 0; w < workers; ++w) buffer.commit_segment(w * seg, seg);
  std::vector<std::thread> th;
  for (size_t w = 0; w < workers; ++w) {
    th.emplace_back([&, w] {
      std::mt19937_64 rng(derive_seed(seed, seed_tag::kCollect, w, 0));
      worker_collect(art.actor, art.critic, *venvs[w], horizon, buffer, w * seg, w * envs_per_worker, rng);
    });
  }
  for (auto& x : th) x.join();
  return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

// VectorizedEnvironment::step alone (env.hpp:200), `threads` VecEnvs of
// envs_per_thread envs each, `steps` steps with U(-1,1) actions.
REF_API double ref_bench_env_step(const double* close, const double* indicators, size_t T, int K, size_t start,
                                  size_t end, size_t threads, size_t envs_per_thread, size_t steps) {
  auto data = make_market(close, indicators, T, K);
  StockConfig cfg;
  EnvFactory factory = [data, cfg, start, end] { return std::make_unique<StockTradingEnv>(data, cfg, start, end); };
  std::vector<std::unique_ptr<VectorizedEnvironment>> venvs;
  std::vector<Tensor2> acts;
  for (size_t w = 0; w < threads; ++w) {
    venvs.push_back(std::make_unique<VectorizedEnvironment>(factory, envs_per_thread));
    venvs[w]->reset(w);
    Tensor2 a(envs_per_thread, K);
    std::mt19937_64 rng(w);
    std::uniform_real_distribution<double> u(-1, 1);
    for (auto& x : a.data) x = u(rng);
    acts.push_back(a);
  }
  auto t0 = std::chrono::steady_clock::now();
  std::vector<std::thread> th;
  for (size_t w = 0; w < threads; ++w)
    th.emplace_back([&, w] {
      for (size_t s = 0; s < steps; ++s) venvs[w]->step(acts[w]);
    });
  for (auto& x : th) x.join();
  return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}
