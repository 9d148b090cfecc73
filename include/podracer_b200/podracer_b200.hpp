// podracer_b200.hpp -- header-only C++ drop-in for the reference's pod hot-path
// API (ElegantRL-podracer, /root/reference/proj/include/podracer), implemented
// over the prb_* C ABI (include/prb.h, libprb.so).
//
// Names, argument meaning, value semantics and exceptions follow the reference:
//   VectorizedEnvironment::reset/step/states/step_counts   env.hpp:167-249
//   policy_sample / policy_mean / gaussian_log_prob         nn.hpp:229-270
//   adam_step                                               nn.hpp:164-182
//   worker_collect + TransitionBuffer                       pod.hpp:95-132, buffer.hpp:27-135
//   buffer_advantages                                       ppo.hpp:212-244
//   ppo_update                                              ppo.hpp:249-296
//   fuse_parameters                                         pod.hpp:141-172
//   leaderboard ranking                                     tournament.hpp:104-119
// Each status code returned by the C ABI is rethrown as the matching
// exception class of common.hpp:19-71.  Host tensors are row-major double,
// exactly the reference's Tensor2 layout; the device keeps fp32 / fp64 copies.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <functional>
#include <memory>
#include <random>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "../prb.h"

namespace podracer_b200 {

// ---- exceptions (common.hpp:19-71) -------------------------------------------
struct DimensionError : std::runtime_error { using std::runtime_error::runtime_error; };
struct NumericError : std::runtime_error { using std::runtime_error::runtime_error; };
struct UsageError : std::runtime_error { using std::runtime_error::runtime_error; };
struct FormatError : std::runtime_error { using std::runtime_error::runtime_error; };
struct DataError : std::runtime_error { using std::runtime_error::runtime_error; };
struct ConfigError : std::runtime_error { using std::runtime_error::runtime_error; };
struct CorruptionError : std::runtime_error { using std::runtime_error::runtime_error; };
struct VersionError : std::runtime_error { using std::runtime_error::runtime_error; };
struct DomainError : std::runtime_error { using std::runtime_error::runtime_error; };
struct DeviceError : std::runtime_error { using std::runtime_error::runtime_error; };

inline void check(int rc) {
  if (rc == PRB_OK) return;
  const std::string m = prb_last_error();
  switch (rc) {
    case PRB_ERR_DIMENSION: throw DimensionError(m);
    case PRB_ERR_NUMERIC: throw NumericError(m);
    case PRB_ERR_USAGE: throw UsageError(m);
    case PRB_ERR_FORMAT: throw FormatError(m);
    case PRB_ERR_DATA: throw DataError(m);
    case PRB_ERR_CONFIG: throw ConfigError(m);
    case PRB_ERR_CORRUPTION: throw CorruptionError(m);
    case PRB_ERR_VERSION: throw VersionError(m);
    case PRB_ERR_DOMAIN: throw DomainError(m);
    default: throw DeviceError(m);
  }
}

// ---- value types mirroring the reference ----------------------------------------
struct Tensor2 {  // tensor.hpp:13-32
  std::size_t rows = 0, cols = 0;
  std::vector<double> data;
  Tensor2() = default;
  Tensor2(std::size_t r, std::size_t c, double fill = 0.0) : rows(r), cols(c), data(r * c, fill) {}
  double& at(std::size_t r, std::size_t c) { return data[r * cols + c]; }
  double at(std::size_t r, std::size_t c) const { return data[r * cols + c]; }
  std::string shape_str() const { return "[" + std::to_string(rows) + "x" + std::to_string(cols) + "]"; }
};

struct StockConfig {  // stock_env.hpp:15-19
  double initial_capital = 1'000'000.0;
  double max_trade_shares = 100.0;
  double cost_rate = 0.002;
};

struct VecStepInfo {  // env.hpp:153-158
  bool episode_end = false;
  std::vector<double> terminal_state;
  double episode_return = 0.0;
  std::size_t episode_length = 0;
};

struct VecStepResult {  // env.hpp:160-165
  Tensor2 next_states;
  std::vector<double> rewards;
  std::vector<std::uint8_t> dones;
  std::vector<VecStepInfo> infos;
};

struct PpoConfig {  // ppo.hpp:18-27
  double gamma = 0.99, gae_lambda = 0.95, clip_eps = 0.2, entropy_coef = 0.01, value_coef = 0.5;
  std::size_t epochs_per_update = 4, minibatch_size = 1024, buffer_size = 4096;
  double learning_rate = 1e-3;
  prb_ppo_config c() const {
    return prb_ppo_config{gamma, gae_lambda, clip_eps, entropy_coef, value_coef, epochs_per_update, minibatch_size,
                          buffer_size, learning_rate};
  }
};

struct PpoUpdateStats {  // ppo.hpp:198-203
  double mean_policy_loss = 0.0, mean_value_loss = 0.0, mean_entropy = 0.0;
  std::size_t minibatches = 0;
};

class Agent;
// ppo.hpp:205-208 (the trained copy lives on the device: a handle instead of a value)
struct PpoUpdateResult {
  std::unique_ptr<Agent> artifact;
  PpoUpdateStats stats;
};

struct PolicySample {  // nn.hpp:245-248
  Tensor2 actions;
  std::vector<double> log_probs;
};

// ---- device handles ------------------------------------------------------------
class Context {
 public:
  explicit Context(int device = 0) { check(prb_ctx_create(device, &h_)); }
  ~Context() { prb_ctx_destroy(h_); }
  Context(const Context&) = delete;
  Context& operator=(const Context&) = delete;
  prb_ctx get() const { return h_; }
  void synchronize() const { check(prb_ctx_synchronize(h_)); }

 private:
  prb_ctx h_ = nullptr;
};

// Device-side MarketData (market.hpp:104-131): close [K][T], indicators [4][K][T].
class MarketData {
 public:
  MarketData(Context& ctx, const std::vector<double>& close, const std::vector<double>* indicators, std::size_t T,
             int K) {
    check(prb_market_create(ctx.get(), close.data(), indicators ? indicators->data() : nullptr, T, K, &h_));
  }
  ~MarketData() { prb_market_destroy(h_); }
  MarketData(const MarketData&) = delete;
  MarketData& operator=(const MarketData&) = delete;
  prb_market get() const { return h_; }

 private:
  prb_market h_ = nullptr;
};

class VectorizedEnvironment {  // env.hpp:167-249
 public:
  static std::unique_ptr<VectorizedEnvironment> stock(const MarketData& m, const StockConfig& cfg, std::size_t start,
                                                      std::size_t end, std::size_t num_envs) {
    prb_stock_config c{cfg.initial_capital, cfg.max_trade_shares, cfg.cost_rate};
    prb_vecenv h = nullptr;
    check(prb_vecenv_create_stock(m.get(), &c, start, end, num_envs, &h));
    return std::unique_ptr<VectorizedEnvironment>(new VectorizedEnvironment(h));
  }
  static std::unique_ptr<VectorizedEnvironment> pointmass(Context& ctx, std::size_t num_envs) {
    prb_vecenv h = nullptr;
    check(prb_vecenv_create_pointmass(ctx.get(), num_envs, &h));
    return std::unique_ptr<VectorizedEnvironment>(new VectorizedEnvironment(h));
  }
  ~VectorizedEnvironment() { prb_vecenv_destroy(h_); }
  VectorizedEnvironment(const VectorizedEnvironment&) = delete;
  VectorizedEnvironment& operator=(const VectorizedEnvironment&) = delete;

  std::size_t num_envs() const { return prb_vecenv_num_envs(h_); }
  const prb_env_spec& spec() const { return spec_; }
  prb_vecenv get() const { return h_; }

  Tensor2 reset(std::uint64_t seed) {
    Tensor2 s(num_envs(), spec_.state_dim);
    check(prb_vecenv_reset_host(h_, seed, s.data.data()));
    return s;
  }
  Tensor2 states() const {
    Tensor2 s(num_envs(), spec_.state_dim);
    check(prb_vecenv_states_host(h_, s.data.data()));
    return s;
  }
  std::vector<std::size_t> step_counts() const {
    std::vector<std::uint64_t> c(num_envs());
    check(prb_vecenv_step_counts_host(h_, c.data()));
    return std::vector<std::size_t>(c.begin(), c.end());
  }
  VecStepResult step(const Tensor2& actions) {
    const std::size_t N = num_envs(), S = spec_.state_dim, A = spec_.action_dim;
    if (actions.rows != N || actions.cols != A)  // env.hpp:201-205
      throw DimensionError("vec_step: actions " + actions.shape_str() + " vs expected [" + std::to_string(N) + "x" +
                           std::to_string(A) + "]");
    VecStepResult out;
    out.next_states = Tensor2(N, S);
    out.rewards.resize(N);
    out.dones.resize(N);
    std::vector<double> term(N * S), tret(N);
    std::vector<std::uint64_t> tlen(N);
    check(prb_vecenv_step_host(h_, actions.data.data(), out.next_states.data.data(), out.rewards.data(),
                               out.dones.data(), term.data(), tret.data(), tlen.data()));
    out.infos.resize(N);
    for (std::size_t i = 0; i < N; ++i) {
      if (!out.dones[i]) continue;
      out.infos[i].episode_end = true;
      out.infos[i].terminal_state.assign(term.begin() + i * S, term.begin() + (i + 1) * S);
      out.infos[i].episode_return = tret[i];
      out.infos[i].episode_length = tlen[i];
    }
    return out;
  }

 private:
  explicit VectorizedEnvironment(prb_vecenv h) : h_(h) { check(prb_vecenv_spec(h_, &spec_)); }
  prb_vecenv h_ = nullptr;
  prb_env_spec spec_{};
};

// Device AgentArtifact: actor (GaussianPolicy) + critic + Adam state in the
// canonical flat layout (artifact.hpp:35-51).
class Agent {
 public:
  Agent(Context& ctx, std::size_t state_dim, std::size_t action_dim, std::vector<std::size_t> hidden = {64, 64})
      : ctx_(&ctx), S_(state_dim), A_(action_dim), hidden_(std::move(hidden)) {
    check(prb_agent_create(ctx.get(), S_, A_, hidden_.data(), (int)hidden_.size(), &h_));
  }
  ~Agent() { prb_agent_destroy(h_); }
  Agent(const Agent&) = delete;
  Agent& operator=(const Agent&) = delete;

  // artifact_init artifact.hpp:91-105 (bit-exact draws)
  static std::unique_ptr<Agent> init(Context& ctx, std::size_t S, std::size_t A, std::uint64_t seed, double lr,
                                     std::vector<std::size_t> hidden = {64, 64}) {
    auto a = std::make_unique<Agent>(ctx, S, A, hidden);
    std::size_t n = 0;
    check(prb_artifact_init(S, A, seed, hidden.data(), (int)hidden.size(), nullptr, &n));
    std::vector<double> flat(n);
    check(prb_artifact_init(S, A, seed, hidden.data(), (int)hidden.size(), flat.data(), nullptr));
    a->set(flat, nullptr, nullptr, 0, lr);
    return a;
  }
  // artifact_init on the device (same mt19937_64 draws, bit-exact; Adam state zeroed): the
  // generator's fresh pods never touch the host (tournament.hpp:142-144)
  void init_device(std::uint64_t seed, double lr) { check(prb_agent_init_device(h_, seed, lr)); }
  // 0: fp32 SIMT update over the whole GPU (default); 1: tensor-core update, one cluster per learner
  void set_ppo_mode(int mode) { check(prb_agent_set_ppo_mode(h_, mode)); }
  std::unique_ptr<Agent> clone() const {
    auto b = std::make_unique<Agent>(*ctx_, S_, A_, hidden_);
    check(prb_agent_copy(b->h_, h_));
    return b;
  }
  std::size_t param_count() const { return prb_agent_param_count(h_); }
  void set(const std::vector<double>& flat, const std::vector<double>* m, const std::vector<double>* v, std::int64_t t,
           double lr) {
    if (flat.size() != param_count())  // unflatten_params artifact.hpp:53-58
      throw DimensionError("unflatten_params: " + std::to_string(flat.size()) + " values vs " +
                           std::to_string(param_count()) + " params");
    check(prb_agent_set_host(h_, flat.data(), m ? m->data() : nullptr, v ? v->data() : nullptr, t, lr));
  }
  std::vector<double> flatten_params() const {
    std::vector<double> f(param_count());
    check(prb_agent_get_host(h_, f.data(), nullptr, nullptr, nullptr));
    return f;
  }
  std::int64_t optimizer_t() const {
    std::int64_t t = 0;
    check(prb_agent_get_host(h_, nullptr, nullptr, nullptr, &t));
    return t;
  }
  void adam_step(const std::vector<double>& grads) {  // nn.hpp:164-182
    if (grads.size() != param_count())
      throw DimensionError("adam_step: params " + std::to_string(param_count()) + ", grads " +
                           std::to_string(grads.size()));
    check(prb_adam_step_host(h_, grads.data()));
  }
  prb_agent get() const { return h_; }
  Context& context() const { return *ctx_; }
  std::size_t state_dim() const { return S_; }
  std::size_t action_dim() const { return A_; }
  const std::vector<std::size_t>& hidden() const { return hidden_; }

 private:
  Context* ctx_;
  std::size_t S_, A_;
  std::vector<std::size_t> hidden_;
  prb_agent h_ = nullptr;
};

namespace detail {
struct DeviceBuffer {
  prb_ctx ctx;
  void* p = nullptr;
  DeviceBuffer(prb_ctx c, std::size_t bytes) : ctx(c) { check(prb_device_alloc(c, bytes, &p)); }
  ~DeviceBuffer() { prb_device_free(ctx, p); }
};
inline std::vector<float> to_f32(const std::vector<double>& v) { return std::vector<float>(v.begin(), v.end()); }
}  // namespace detail

// policy_sample nn.hpp:250-265 (noise: Philox stream keyed by seed/counter)
inline PolicySample policy_sample(const Agent& a, const Tensor2& states, std::uint64_t seed, std::uint64_t counter = 0) {
  if (states.cols != a.state_dim())
    throw DimensionError("mlp_forward: input " + states.shape_str() + " vs weights [" + std::to_string(a.state_dim()) +
                         "x..]");
  prb_ctx c = a.context().get();
  const std::size_t n = states.rows, A = a.action_dim();
  detail::DeviceBuffer ds(c, n * states.cols * 4 + 4), da(c, n * A * 4 + 4), dl(c, n * 4 + 4);
  const std::vector<float> s32 = detail::to_f32(states.data);
  check(prb_memcpy_h2d(c, ds.p, s32.data(), s32.size() * 4));
  check(prb_policy_sample(a.get(), static_cast<const float*>(ds.p), n, seed, counter, static_cast<float*>(da.p),
                          static_cast<float*>(dl.p), nullptr, nullptr));
  std::vector<float> act(n * A), lp(n);
  check(prb_memcpy_d2h(c, act.data(), da.p, act.size() * 4));
  check(prb_memcpy_d2h(c, lp.data(), dl.p, lp.size() * 4));
  PolicySample out;
  out.actions = Tensor2(n, A);
  out.actions.data.assign(act.begin(), act.end());
  out.log_probs.assign(lp.begin(), lp.end());
  return out;
}

// The reference's signature (nn.hpp:250): the noise is Philox keyed by ONE 64-bit draw of rng.
inline PolicySample policy_sample(const Agent& a, const Tensor2& states, std::mt19937_64& rng) {
  return policy_sample(a, states, rng(), 0);
}

// Device TransitionBuffer sized for one VecEnv x horizon (buffer.hpp:39-48).
class TransitionBuffer {
 public:
  TransitionBuffer(const VectorizedEnvironment& env, std::size_t horizon) {
    check(prb_rollout_create(env.get(), horizon, &h_));
    N_ = env.num_envs();
    H_ = horizon;
    S_ = env.spec().state_dim;
    A_ = env.spec().action_dim;
  }
  ~TransitionBuffer() { prb_rollout_destroy(h_); }
  TransitionBuffer(const TransitionBuffer&) = delete;
  TransitionBuffer& operator=(const TransitionBuffer&) = delete;
  std::size_t capacity() const { return N_ * H_; }
  std::size_t length() const { return N_ * H_; }  // a collect fills the whole buffer
  bool full() const { return true; }
  std::size_t horizon() const { return H_; }
  std::size_t num_envs() const { return N_; }
  prb_rollout get() const { return h_; }
  // Host copies of the columns in the reference index space (env e, step t at e*H + t,
  // pod.hpp:89-94); the reference returns references to its host vectors (buffer.hpp:55-61),
  // here each call downloads the device column.
  std::vector<double> states() const { return column(0, S_); }
  std::vector<double> actions() const { return column(1, A_); }
  std::vector<double> log_probs() const { return column(2, 1); }
  std::vector<double> rewards() const { return column(3, 1); }
  std::vector<double> values() const { return column(5, 1); }
  std::vector<std::uint8_t> dones() const {
    std::vector<std::uint8_t> d(capacity());
    check(prb_rollout_download(h_, nullptr, nullptr, nullptr, nullptr, d.data(), nullptr, nullptr));
    return d;
  }
  std::vector<double> bootstrap_values() const {  // Chunk::bootstrap_value of env e's chunk
    std::vector<double> b(N_);
    check(prb_rollout_download(h_, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, b.data()));
    return b;
  }
  std::size_t state_dim() const { return S_; }
  std::size_t action_dim() const { return A_; }

 private:
  std::vector<double> column(int which, std::size_t width) const {
    std::vector<double> v(capacity() * width);
    double* p[6] = {nullptr, nullptr, nullptr, nullptr, nullptr, nullptr};
    p[which] = v.data();
    check(prb_rollout_download(h_, p[0], p[1], p[2], p[3], nullptr, p[5], nullptr));
    return v;
  }
  prb_rollout h_ = nullptr;
  std::size_t N_ = 0, H_ = 0, S_ = 0, A_ = 0;
};

// worker_collect pod.hpp:95-132
inline void worker_collect(const Agent& a, VectorizedEnvironment& env, TransitionBuffer& buf, std::uint64_t seed) {
  check(prb_rollout_collect(buf.get(), a.get(), env.get(), seed));
}

// The reference's signature (pod.hpp:95-98): the actor and critic are the agent's; the noise is
// Philox keyed by ONE 64-bit draw of the caller's rng (the reference draws N x A x H normals from
// it, so the caller's stream advances differently; both are deterministic in the seed).  The
// device buffer holds one VecEnv's segment: segment_offset and chunk_base must be 0 and horizon
// the buffer's (a multi-worker pod_train uses one VecEnv of num_workers * envs_per_worker envs).
inline void worker_collect(const Agent& a, VectorizedEnvironment& env, std::size_t horizon, TransitionBuffer& buf,
                           std::size_t segment_offset, std::size_t chunk_base, std::mt19937_64& rng) {
  if (segment_offset != 0 || chunk_base != 0 || horizon != buf.horizon() || env.num_envs() != buf.num_envs())
    throw UsageError("worker_collect: the device buffer holds one VecEnv's segment (offset 0, chunk base 0, its "
                     "horizon and env count)");
  worker_collect(a, env, buf, rng());
}

// worker_collect of every pod of a GPU in ONE launch (per-pod weights, buffers and seeds);
// identical to P worker_collect calls
inline void worker_collect_pods(const std::vector<const Agent*>& agents, const std::vector<VectorizedEnvironment*>& envs,
                                const std::vector<TransitionBuffer*>& bufs, const std::vector<std::uint64_t>& seeds) {
  const std::size_t P = agents.size();
  if (envs.size() != P || bufs.size() != P || seeds.size() != P)
    throw DimensionError("worker_collect_pods: " + std::to_string(P) + " agents, " + std::to_string(envs.size()) +
                         " envs, " + std::to_string(bufs.size()) + " buffers, " + std::to_string(seeds.size()) +
                         " seeds");
  std::vector<prb_rollout> r(P);
  std::vector<prb_agent> a(P);
  std::vector<prb_vecenv> e(P);
  for (std::size_t p = 0; p < P; ++p) {
    r[p] = bufs[p]->get();
    a[p] = agents[p]->get();
    e[p] = envs[p]->get();
  }
  check(prb_rollout_collect_pods(r.data(), a.data(), e.data(), P, seeds.data()));
}

// buffer_advantages ppo.hpp:212-244 -> (advantages, returns), reference index space
inline std::pair<std::vector<double>, std::vector<double>> buffer_advantages(TransitionBuffer& buf,
                                                                             const PpoConfig& cfg,
                                                                             bool normalize = true) {
  check(prb_gae(buf.get(), cfg.gamma, cfg.gae_lambda, normalize ? 1 : 0));
  std::vector<double> adv(buf.capacity()), ret(buf.capacity());
  check(prb_gae_download(buf.get(), adv.data(), ret.data()));
  return {std::move(adv), std::move(ret)};
}

// ppo_update ppo.hpp:249-296: returns a trained copy (.artifact) and its statistics (.stats);
// the input is untouched.
inline PpoUpdateResult ppo_update(const Agent& a, TransitionBuffer& buf, const PpoConfig& cfg, std::uint64_t seed,
                                  const std::vector<std::uint64_t>* perm = nullptr) {
  auto out = std::make_unique<Agent>(a.context(), a.state_dim(), a.action_dim(), a.hidden());
  const prb_ppo_config c = cfg.c();
  prb_ppo_stats st{};
  check(prb_ppo_update(a.get(), buf.get(), &c, seed, perm ? perm->data() : nullptr, out->get(), &st));
  return {std::move(out), PpoUpdateStats{st.mean_policy_loss, st.mean_value_loss, st.mean_entropy, st.minibatches}};
}

// The learner phase of pod_train (pod.hpp:436-461): learner l = ppo_update(*agents[l], *bufs[l],
// cfg, seeds[l]); all learners in ONE tensor-core launch (a thread-block cluster each).
inline std::pair<std::vector<std::unique_ptr<Agent>>, std::vector<PpoUpdateStats>> ppo_update_learners(
    const std::vector<const Agent*>& agents, const std::vector<TransitionBuffer*>& bufs, const PpoConfig& cfg,
    const std::vector<std::uint64_t>& seeds) {
  const std::size_t L = agents.size();
  if (bufs.size() != L || seeds.size() != L)
    throw DimensionError("ppo_update_learners: " + std::to_string(L) + " agents, " + std::to_string(bufs.size()) +
                         " buffers, " + std::to_string(seeds.size()) + " seeds");
  std::vector<std::unique_ptr<Agent>> outs;
  std::vector<prb_agent> src(L), dst(L);
  std::vector<prb_rollout> r(L);
  for (std::size_t l = 0; l < L; ++l) {
    const Agent& a = *agents[l];
    outs.push_back(std::make_unique<Agent>(a.context(), a.state_dim(), a.action_dim(), a.hidden()));
    src[l] = a.get();
    dst[l] = outs.back()->get();
    r[l] = bufs[l]->get();
  }
  const prb_ppo_config c = cfg.c();
  std::vector<prb_ppo_stats> st(L);
  check(prb_ppo_update_learners(src.data(), r.data(), L, &c, seeds.data(), dst.data(), st.data()));
  std::vector<PpoUpdateStats> stats;
  for (const auto& x : st) stats.push_back(PpoUpdateStats{x.mean_policy_loss, x.mean_value_loss, x.mean_entropy,
                                                          x.minibatches});
  return {std::move(outs), std::move(stats)};
}

// save_checkpoint / load_checkpoint checkpoint.hpp:305-317 (PODRCKPT v1, the reference's bytes)
inline void save_checkpoint(const Agent& a, const std::string& path, std::int64_t parent_pod = -1,
                            std::uint64_t mutation_seed = 0, const std::string& algo_tag = "ppo") {
  check(prb_checkpoint_save(a.get(), path.c_str(), parent_pod, mutation_seed, algo_tag.c_str(), nullptr));
}
struct CheckpointInfo {
  std::int64_t parent_pod = -1;
  std::uint64_t mutation_seed = 0;
  std::string algo_tag;
};
inline CheckpointInfo load_checkpoint(Agent& a, const std::string& path) {
  CheckpointInfo info;
  char tag[256] = {0};
  int has_meta = 0;
  double meta[3];
  check(prb_checkpoint_load(a.get(), path.c_str(), &info.parent_pod, &info.mutation_seed, tag, sizeof(tag), meta,
                            &has_meta));
  info.algo_tag = tag;
  return info;
}

// EvaluationRecord pod.hpp:30-36 and evaluate pod.hpp:43-83: one episode per env of
// `env` (reset with derive_seed(seed, kEpisode, i); its state is consumed).
struct EvaluationRecord {
  double wall_seconds = 0.0;
  std::int64_t env_steps = 0;
  std::vector<double> episodic_rewards;
  double mean = 0.0;
  double std_dev = 0.0;
  std::uint64_t eval_steps = 0;
};

inline EvaluationRecord evaluate(const Agent& actor, VectorizedEnvironment& env, std::uint64_t seed,
                                 bool sample_actions = false) {
  EvaluationRecord rec;
  rec.episodic_rewards.resize(env.num_envs());
  check(prb_evaluate(actor.get(), env.get(), seed, sample_actions ? 1 : 0, rec.episodic_rewards.data(), &rec.mean,
                     &rec.std_dev, &rec.eval_steps));
  return rec;
}

// evaluate for every pod of a GPU in one pass (record p == evaluate(*agents[p], *envs[p], seeds[p]))
inline std::vector<EvaluationRecord> evaluate_pods(const std::vector<const Agent*>& agents,
                                                   const std::vector<VectorizedEnvironment*>& envs,
                                                   const std::vector<std::uint64_t>& seeds, bool sample_actions = false) {
  const std::size_t P = agents.size();
  if (envs.size() != P || seeds.size() != P)
    throw DimensionError("evaluate_pods: " + std::to_string(P) + " agents, " + std::to_string(envs.size()) +
                         " envs, " + std::to_string(seeds.size()) + " seeds");
  if (P == 0) return {};
  const std::size_t n = envs[0]->num_envs();
  std::vector<prb_agent> a(P);
  std::vector<prb_vecenv> e(P);
  for (std::size_t p = 0; p < P; ++p) {
    a[p] = agents[p]->get();
    e[p] = envs[p]->get();
  }
  std::vector<double> r(P * n), m(P), sd(P);
  std::vector<std::uint64_t> st(P);
  check(prb_evaluate_pods(a.data(), e.data(), P, seeds.data(), sample_actions ? 1 : 0, r.data(), m.data(), sd.data(),
                          st.data()));
  std::vector<EvaluationRecord> out(P);
  for (std::size_t p = 0; p < P; ++p) {
    out[p].episodic_rewards.assign(r.begin() + p * n, r.begin() + (p + 1) * n);
    out[p].mean = m[p];
    out[p].std_dev = sd[p];
    out[p].eval_steps = st[p];
  }
  return out;
}

// fuse_parameters pod.hpp:141-172
inline std::unique_ptr<Agent> fuse_parameters(const std::vector<const Agent*>& agents) {
  if (agents.empty()) throw UsageError("fuse_parameters: empty artifact list");
  const Agent& a0 = *agents.front();
  auto out = std::make_unique<Agent>(a0.context(), a0.state_dim(), a0.action_dim(), a0.hidden());
  std::vector<prb_agent> hs;
  for (const Agent* a : agents) hs.push_back(a->get());
  check(prb_fuse_parameters(hs.data(), hs.size(), out->get()));
  return out;
}

// Leaderboard order after inserting candidates in seq order (tournament.hpp:104-119)
inline std::vector<int> leaderboard_rank(Context& ctx, const std::vector<double>& scores,
                                         const std::vector<std::uint64_t>& seqs, std::size_t capacity) {
  std::vector<std::int32_t> order(capacity);
  std::int32_t n = 0;
  check(prb_leaderboard_rank_host(ctx.get(), scores.data(), seqs.data(), scores.size(), capacity, order.data(), &n));
  return std::vector<int>(order.begin(), order.begin() + n);
}

// ---- Leaderboard tournament.hpp:31-119 -----------------------------------------
// Entries keep their agents on the device; refresh_stats runs prb_leaderboard_stats over the
// entries' parameter blobs (fp64, the reference's summation order).
struct PopulationStats {  // tournament.hpp:38-41
  std::vector<double> mean;
  std::vector<double> variance;
};

struct LeaderboardEntry {  // tournament.hpp:31-36
  std::shared_ptr<const Agent> artifact;
  double score = 0.0;
  std::int64_t pod_id = -1;
  std::uint64_t seq = 0;
};

class Leaderboard {
 public:
  explicit Leaderboard(std::size_t capacity = 10) : capacity_(capacity) {
    if (capacity_ == 0) throw ConfigError("Leaderboard: capacity must be > 0");
  }
  std::size_t capacity() const { return capacity_; }
  std::size_t size() const { return entries_.size(); }
  bool empty() const { return entries_.empty(); }
  const std::vector<LeaderboardEntry>& entries() const { return entries_; }
  const LeaderboardEntry& at(std::size_t rank) const { return entries_.at(rank); }
  const PopulationStats& stats() const { return stats_; }
  double min_score() const { return entries_.back().score; }
  double best_score() const { return entries_.front().score; }
  std::uint64_t next_seq() { return seq_counter_++; }
  std::vector<LeaderboardEntry>& mutable_entries() { return entries_; }
  void refresh_stats() {  // tournament.hpp:66-87, on the device
    stats_.mean.clear();
    stats_.variance.clear();
    if (entries_.empty()) return;
    std::vector<prb_agent> hs;
    for (const auto& e : entries_) hs.push_back(e.artifact->get());
    const std::size_t P = entries_.front().artifact->param_count();
    stats_.mean.assign(P, 0.0);
    stats_.variance.assign(P, 0.0);
    check(prb_leaderboard_stats_host(hs.data(), hs.size(), stats_.mean.data(), stats_.variance.data()));
  }

 private:
  std::size_t capacity_;
  std::vector<LeaderboardEntry> entries_;  // (score desc, seq asc)
  PopulationStats stats_;
  std::uint64_t seq_counter_ = 0;
};

struct LeaderboardUpdate {  // tournament.hpp:93-96
  bool inserted = false;
  bool has_rank = false;
  std::size_t rank = 0;
};

// leaderboard_update tournament.hpp:104-119: non-finite -> NumericError; seq = arrival counter;
// a full board rejects scores <= its minimum; insert after every entry scoring >= the candidate;
// evict the tail; refresh the population stats.
inline LeaderboardUpdate leaderboard_update(Leaderboard& board, LeaderboardEntry candidate) {
  if (!(candidate.score == candidate.score) || candidate.score == HUGE_VAL || candidate.score == -HUGE_VAL)
    throw NumericError("leaderboard_update: candidate score is not finite");
  candidate.seq = board.next_seq();
  auto& entries = board.mutable_entries();
  if (entries.size() >= board.capacity() && candidate.score <= entries.back().score) return {};
  std::size_t pos = 0;
  while (pos < entries.size() && entries[pos].score >= candidate.score) ++pos;
  entries.insert(entries.begin() + (std::ptrdiff_t)pos, std::move(candidate));
  if (entries.size() > board.capacity()) entries.pop_back();
  board.refresh_stats();
  return LeaderboardUpdate{true, true, pos};
}

// GeneratorConfig tournament.hpp:125-129
struct GeneratorConfig {
  std::size_t top_k = 3;
  double mutation_sigma = 0.01;
  double fresh_prob = 0.2;
};

struct PodLineage {  // the AgentArtifact::lineage fields generate_pod_init sets
  std::int64_t parent_pod = -1;
  std::uint64_t mutation_seed = 0;
};

// generate_pod_init tournament.hpp:136-162.  `board` is the leaderboard's entries in rank order
// (their agents stay on the device); the fresh / parent decision consumes the caller's
// mt19937_64 exactly as the reference does (same libstdc++ distributions, same draw order:
// u01, pick, mutation seed), so a pod_train driver makes the same choices; the copy and the
// mutation never leave HBM: prb_agent_copy, then prb_agent_mutate (params += N(0, sigma^2) from a
// Philox stream keyed by the reference's mutation seed -- statistics-level parity, DESIGN.md §6 --
// and optimizer t := 0 with m / v kept).
inline std::unique_ptr<Agent> generate_pod_init(const std::vector<const Agent*>& board,
                                                const std::vector<std::int64_t>& board_pod_ids,
                                                const GeneratorConfig& cfg, std::mt19937_64& rng,
                                                const std::function<std::unique_ptr<Agent>(std::uint64_t)>& fresh_init,
                                                PodLineage* lineage = nullptr) {
  if (cfg.top_k < 1) throw ConfigError("generator.top_k must be >= 1");
  if (board_pod_ids.size() != board.size())
    throw DimensionError("generate_pod_init: " + std::to_string(board.size()) + " entries, " +
                         std::to_string(board_pod_ids.size()) + " pod ids");
  std::uniform_real_distribution<double> u01(0.0, 1.0);
  if (board.empty() || u01(rng) < cfg.fresh_prob) {
    auto fresh = fresh_init(rng());
    if (lineage) *lineage = PodLineage{};
    return fresh;
  }
  const std::size_t pool = std::min(cfg.top_k, board.size());
  std::uniform_int_distribution<std::size_t> pick(0, pool - 1);
  const std::size_t i = pick(rng);
  auto child = board.at(i)->clone();
  const std::uint64_t mseed = rng();
  if (lineage) *lineage = PodLineage{board_pod_ids[i], mseed};
  check(prb_agent_mutate(child->get(), mseed, cfg.mutation_sigma > 0.0 ? cfg.mutation_sigma : 0.0));
  return child;
}

}  // namespace podracer_b200
