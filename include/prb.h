/*
 * prb.h -- C ABI of the B200-native pod hot path (podracer-b200).
 *
 * The reference (ElegantRL-podracer restated as header-only C++20 under
 * /root/reference/proj/include/podracer) has no C ABI; its "operator API" is
 * a set of value-semantic C++ functions that throw.  Each
 * prb_* entry point below replaces one of them; the comment on each names the
 * reference interface (file:line) it stands in for.  include/podracer_b200/
 * podracer_b200.hpp re-exposes these with the reference's C++ signatures.
 *
 * Conventions
 *   - Plain pointers and sizes only.  `d_` pointers are device (cuda:N)
 *     pointers; everything else is host memory.  Device work is issued on
 *     the context's stream; functions that return host data synchronise it.
 *   - Every function returns an int status: 0 = PRB_OK, otherwise the
 *     PRB_ERR_* code of the reference exception class it mirrors
 *     (common.hpp:19-71).  prb_last_error() gives the message (thread-local).
 *   - Validation happens before any state changes, as in the reference
 *     (e.g. adam_step nn.hpp:162-171).
 *   - Reals on the device are fp32 except the stock portfolio accounting
 *     (balance, rewards before storage, episode returns), which is fp64 so
 *     integer share decisions stay bit-exact.
 */
#ifndef PRB_H_
#define PRB_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PRB_API __attribute__((visibility("default")))

/* Status codes == reference exception classes (common.hpp:19-71). */
#define PRB_OK 0
#define PRB_ERR_DIMENSION 1  /* DimensionError  common.hpp:20 */
#define PRB_ERR_NUMERIC 2    /* NumericError    common.hpp:26 */
#define PRB_ERR_USAGE 3      /* UsageError      common.hpp:32 */
#define PRB_ERR_FORMAT 4     /* FormatError     common.hpp:38 */
#define PRB_ERR_DATA 5       /* DataError       common.hpp:44 */
#define PRB_ERR_CONFIG 6     /* ConfigError     common.hpp:50 */
#define PRB_ERR_CORRUPTION 7 /* CorruptionError common.hpp:56 */
#define PRB_ERR_VERSION 8    /* VersionError    common.hpp:62 */
#define PRB_ERR_DOMAIN 9     /* DomainError     common.hpp:69 */
#define PRB_ERR_CUDA 10      /* device / driver failure (no reference analogue) */

PRB_API const char* prb_last_error(void);
PRB_API int prb_version(void);

/* ---- seeds: common.hpp:79-105 ------------------------------------------ */
PRB_API uint64_t prb_splitmix64(uint64_t x);                                   /* common.hpp:79 */
PRB_API uint64_t prb_derive_seed(uint64_t base, const uint64_t* tags, int n);  /* common.hpp:88 */

/* ---- context: one device + one stream (the reference's worker thread) ---- */
typedef struct prb_ctx_s* prb_ctx;
PRB_API int prb_ctx_create(int device, prb_ctx* out);
PRB_API int prb_ctx_destroy(prb_ctx ctx);
PRB_API int prb_ctx_synchronize(prb_ctx ctx);
PRB_API void* prb_ctx_stream(prb_ctx ctx); /* cudaStream_t */
PRB_API int prb_device_alloc(prb_ctx ctx, size_t bytes, void** d_out);
PRB_API int prb_device_free(prb_ctx ctx, void* d_ptr);
PRB_API int prb_memcpy_h2d(prb_ctx ctx, void* d_dst, const void* src, size_t bytes); /* synchronous */
PRB_API int prb_memcpy_d2h(prb_ctx ctx, void* dst, const void* d_src, size_t bytes); /* synchronous */
PRB_API int prb_memcpy_h2d_async(prb_ctx ctx, void* d_dst, const void* src, size_t bytes);
PRB_API int prb_memcpy_d2h_async(prb_ctx ctx, void* dst, const void* d_src, size_t bytes);
/* Per-kernel CUDA-event timing on the context's stream (no reference
 * analogue; the reference has no tracing).  enable resets the
 * counters; read returns the summed device milliseconds and launch count of
 * one kernel class. */
#define PRB_PROF_POLICY 0
#define PRB_PROF_ENV_STOCK 1
#define PRB_PROF_ENV_POINTMASS 2
#define PRB_PROF_GAE 3
#define PRB_PROF_PPO_FWDBWD 4
#define PRB_PROF_PPO_REDUCE 5
#define PRB_PROF_ADAM 6
#define PRB_PROF_ROLLOUT 7
PRB_API int prb_ctx_profile(prb_ctx ctx, int enable);
PRB_API int prb_ctx_profile_read(prb_ctx ctx, int kind, double* total_ms, uint64_t* launches);

/* ---- market data (market.hpp) ------------------------------------------ */
/* Synthetic OHLCV of BASELINE.md §3: mt19937_64(seed); p0 ~ U(10,200);
 * p_{t+1} = p_t * exp(1e-3 N(0,1)); open=close, high=1.001p, low=0.999p,
 * volume=1000.  Arrays are [K][T]; any output may be NULL. */
PRB_API int prb_market_synthetic(uint64_t seed, int K, size_t T, double* open, double* high, double* low,
                                 double* close, double* volume);
/* compute_indicators market.hpp:373-392 (MACD, RSI-14, CCI-30, SMA-20);
 * out[(i*K + k)*T + t].  DataError when T < 35. */
PRB_API int prb_compute_indicators(const double* high, const double* low, const double* close, size_t T, int K,
                                   double* out);

typedef struct prb_market_s* prb_market;
/* MarketData (market.hpp:104-131) after compute_indicators: close [K][T],
 * indicators [4][K][T] (kIndicatorNames order, market.hpp:101). */
PRB_API int prb_market_create(prb_ctx ctx, const double* close, const double* indicators, size_t T, int K,
                              prb_market* out);
PRB_API int prb_market_destroy(prb_market m);

/* ---- vectorised environments (env.hpp:167-249) ------------------------- */
typedef struct {
  double initial_capital;  /* StockConfig stock_env.hpp:15-19 */
  double max_trade_shares;
  double cost_rate;
} prb_stock_config;

typedef struct {
  size_t state_dim, action_dim, max_episode_steps; /* EnvSpec env.hpp:16-34 */
  double reward_target;
  const double* action_low;  /* action_dim entries, owned by the env */
  const double* action_high;
} prb_env_spec;

typedef struct prb_vecenv_s* prb_vecenv;
/* VectorizedEnvironment(factory -> StockTradingEnv(data, cfg, start, end), N)
 * env.hpp:169 + stock_env.hpp:137-154 (validation: UsageError without
 * indicators, ConfigError on a bad window, ConfigError on N == 0). */
PRB_API int prb_vecenv_create_stock(prb_market m, const prb_stock_config* cfg, size_t start, size_t end,
                                    size_t num_envs, prb_vecenv* out);
/* VectorizedEnvironment(factory -> PointMass2D, N) env.hpp:111-146. */
PRB_API int prb_vecenv_create_pointmass(prb_ctx ctx, size_t num_envs, prb_vecenv* out);
PRB_API int prb_vecenv_destroy(prb_vecenv env);
PRB_API int prb_vecenv_spec(prb_vecenv env, prb_env_spec* out);   /* spec() env.hpp:181 */
PRB_API size_t prb_vecenv_num_envs(prb_vecenv env);                /* num_envs() env.hpp:180 */
PRB_API const float* prb_vecenv_states_device(prb_vecenv env);     /* states() env.hpp:182, [N][S] fp32 */
/* reset(seed) env.hpp:186-194.  Per-env streams derive_seed(seed, kVecEnv, i)
 * (mt19937_64, bit-exact with the reference).  d_obs (nullable) receives [N][S]. */
PRB_API int prb_vecenv_reset(prb_vecenv env, uint64_t seed, float* d_obs);
/* step(actions) env.hpp:200-236 on device buffers.  d_actions [N][A] fp32
 * (unclipped; clipped to the spec bounds inside).  Outputs (each nullable):
 * d_reward [N], d_done [N], and for rows that ended an episode only:
 * d_terminal_obs [N][S], d_episode_return [N] (fp64), d_episode_length [N].
 * The new states (post auto-reset) land in prb_vecenv_states_device(). */
PRB_API int prb_vecenv_step(prb_vecenv env, const float* d_actions, float* d_reward, uint8_t* d_done,
                            float* d_terminal_obs, double* d_episode_return, int32_t* d_episode_length);
/* Host-buffer forms with the reference's Tensor2 (double) layouts. */
PRB_API int prb_vecenv_reset_host(prb_vecenv env, uint64_t seed, double* states);
PRB_API int prb_vecenv_step_host(prb_vecenv env, const double* actions, double* next_states, double* rewards,
                                 uint8_t* dones, double* terminal_states, double* episode_returns,
                                 uint64_t* episode_lengths);
PRB_API int prb_vecenv_states_host(prb_vecenv env, double* states);
PRB_API int prb_vecenv_step_counts_host(prb_vecenv env, uint64_t* out); /* step_counts() env.hpp:183 */

/* ---- agent: actor (GaussianPolicy) + critic + Adam ---------------------- */
typedef struct prb_agent_s* prb_agent;
/* AgentArtifact shape (artifact.hpp:23-86): actor S->hidden...->A (tanh
 * hidden, linear out, nn.hpp:63-85), log_std[A], critic S->hidden...->1. */
PRB_API int prb_agent_create(prb_ctx ctx, size_t state_dim, size_t action_dim, const size_t* hidden, int n_hidden,
                             prb_agent* out);
PRB_API int prb_agent_destroy(prb_agent a);
PRB_API size_t prb_agent_param_count(prb_agent a);                  /* param_count() artifact.hpp:30 */
/* flatten/unflatten_params artifact.hpp:38-72 + AdamState nn.hpp:144-152.
 * m/v may be NULL (zeros on set, skipped on get). */
PRB_API int prb_agent_set_host(prb_agent a, const double* flat, const double* m, const double* v, int64_t t,
                               double lr);
PRB_API int prb_agent_get_host(prb_agent a, double* flat, double* m, double* v, int64_t* t);
PRB_API int prb_agent_copy(prb_agent dst, prb_agent src); /* AgentArtifact copy (deep) */
PRB_API float* prb_agent_params_device(prb_agent a);       /* [P] fp32 flat blob */
/* artifact_init artifact.hpp:91-105 ON THE DEVICE into agent a (its shapes):
 * the reference's mt19937_64 streams and uniform_real_distribution draw order
 * (nn.hpp:40-54), so the fp32 params are the reference's values rounded once;
 * Adam state zero, learning rate lr.  The generator's fresh pods never touch
 * the host (tournament.hpp:142-144). */
PRB_API int prb_agent_init_device(prb_agent a, uint64_t seed, double lr);
/* artifact_init artifact.hpp:91-105 (host, bit-exact with the reference). */
PRB_API int prb_artifact_init(size_t state_dim, size_t action_dim, uint64_t seed, const size_t* hidden, int n_hidden,
                              double* flat_out, size_t* param_count);

/* ---- policy (nn.hpp:229-277) -------------------------------------------- */
/* policy_sample nn.hpp:250-265 fused with the critic forward of worker_collect
 * (pod.hpp:112-113).  Noise: Philox4x32-10 keyed by (seed), counter =
 * (counter, row, d).  d_values / d_eps nullable; d_eps receives the unit
 * normals used (parity seam).  NumericError on non-finite states. */
PRB_API int prb_policy_sample(prb_agent a, const float* d_states, size_t n, uint64_t seed, uint64_t counter,
                              float* d_actions, float* d_log_probs, float* d_values, float* d_eps);
/* Same with injected unit normals d_eps [n][A] (reference-side seam). */
PRB_API int prb_policy_sample_eps(prb_agent a, const float* d_states, size_t n, const float* d_eps,
                                  float* d_actions, float* d_log_probs, float* d_values);
PRB_API int prb_policy_mean(prb_agent a, const float* d_states, size_t n, float* d_mean);        /* nn.hpp:268 */
PRB_API int prb_policy_log_prob(prb_agent a, const float* d_states, const float* d_actions, size_t n,
                                float* d_log_probs);                                              /* nn.hpp:229 */
PRB_API int prb_critic_value(prb_agent a, const float* d_states, size_t n, float* d_values);      /* nn.hpp:63 */

/* ---- rollout buffer + collection (buffer.hpp, pod.hpp:95-132) ----------- */
typedef struct prb_rollout_s* prb_rollout;
/* TransitionBuffer(N*H, S, A) buffer.hpp:39-48, sized for one VecEnv of N
 * envs collected for H steps.  The stock env's rows are stored compactly
 * (balance/cap + shares per transition, the 150 shared features by time
 * index); other envs store full rows. */
PRB_API int prb_rollout_create(prb_vecenv env, size_t horizon, prb_rollout* out);
/* As above for an externally supplied buffer (full rows, no env). */
PRB_API int prb_rollout_create_raw(prb_ctx ctx, size_t num_envs, size_t horizon, size_t state_dim, size_t action_dim,
                                   prb_rollout* out);
PRB_API int prb_rollout_destroy(prb_rollout r);
/* worker_collect pod.hpp:95-132: H steps of policy_sample + critic + step,
 * then the bootstrap V(s_H) per env.  Noise stream keyed by seed (the
 * reference's derive_seed(seed, kCollect, w, epoch)). */
PRB_API int prb_rollout_collect(prb_rollout r, prb_agent a, prb_vecenv env, uint64_t seed);
/* worker_collect of P pods at once (all pods of a GPU in
 * ONE launch, per-pod weights as a grouped GEMM): rollout p = worker_collect(
 * agents[p], envs[p]) with noise seed seeds[p], exactly what P separate
 * prb_rollout_collect calls in mode 2 compute, when every pod is a stock VecEnv
 * on the tcgen05 path (64x64 nets) with the same num_envs, horizon and asset
 * count; other pods (e.g. PointMass) are collected one by one.  Rollouts and
 * VecEnvs distinct. */
PRB_API int prb_rollout_collect_pods(const prb_rollout* rollouts, const prb_agent* agents, const prb_vecenv* envs,
                                     size_t P, const uint64_t* seeds);
/* Collection mode.  When the shapes allow it (stock env, 64x64 nets):
 * 2 (default) = one fused persistent kernel per rollout, actor/critic layers
 * on tcgen05 tensor cores (bf16 operands, fp32 TMEM accumulators);
 * 1 = the same fused kernel with fp32 SIMT layers (reference-precision path).
 * 0 = one policy launch + one VecEnv step launch per time step (the kernels
 * prb_policy_sample / prb_vecenv_step run).  Other shapes always use 0. */
PRB_API int prb_rollout_set_mode(prb_rollout r, int mode);
/* Device views of the time-major buffer fields ([H][N] rows; obs rows hold
 * the stored obs floats per transition). Any out pointer may be NULL. */
PRB_API int prb_rollout_device_fields(prb_rollout r, float** d_obs, float** d_actions, float** d_log_probs,
                                      float** d_rewards, float** d_values, uint8_t** d_dones, float** d_bootstrap);
/* Host transfer in the REFERENCE index space (chunk e = rows e*H..e*H+H-1,
 * pod.hpp:89-94): states [N*H][S], actions [N*H][A], log_probs, rewards,
 * dones, values [N*H], bootstrap [N].  Any pointer may be NULL (download). */
PRB_API int prb_rollout_download(prb_rollout r, double* states, double* actions, double* log_probs, double* rewards,
                                 uint8_t* dones, double* values, double* bootstrap);
/* The chunks of selected envs only (TransitionBuffer rows e*H .. e*H+H-1 of
 * each env e = envs[i], pod.hpp:89-94), written as chunk i = rows i*H ..
 * i*H+H-1 of the outputs; bootstrap [n_envs].  raw_advantages / returns are
 * the un-normalised GAE outputs of the last prb_gae (ppo.hpp:50-71; the
 * normalisation is prb_gae_stats).  Any pointer may be NULL. */
PRB_API int prb_rollout_download_chunks(prb_rollout r, const uint64_t* envs, size_t n_envs, double* states,
                                        double* actions, double* log_probs, double* rewards, uint8_t* dones,
                                        double* values, double* bootstrap, double* raw_advantages, double* returns);
PRB_API int prb_rollout_upload(prb_rollout r, const double* states, const double* actions, const double* log_probs,
                               const double* rewards, const uint8_t* dones, const double* values,
                               const double* bootstrap);

/* ---- GAE (ppo.hpp:50-71, 212-244) --------------------------------------- */
/* buffer_advantages: per-env reverse scan + whole-buffer mean/std (std floor
 * 1e-8).  Results stay on device for prb_ppo_update. */
PRB_API int prb_gae(prb_rollout r, double gamma, double lambda, int normalize);
/* Normalised advantages and returns in the reference index space. */
PRB_API int prb_gae_download(prb_rollout r, double* advantages, double* returns);
/* The whole-buffer advantage normalisation of the last prb_gae
 * (buffer_advantages ppo.hpp:234-242): normalised = (raw - mean) / denom,
 * denom = max(population std, 1e-8); (0, 1) when normalize was 0. */
PRB_API int prb_gae_stats(prb_rollout r, double* mean, double* denom);
/* Seam: set the (already normalised) advantages and returns directly, in the
 * reference index space -- the inputs gather_minibatch (ppo.hpp:83-103) reads. */
PRB_API int prb_rollout_set_advantages(prb_rollout r, const double* advantages, const double* returns);
/* compute_gae over raw device arrays in TIME-MAJOR layout [H][N]. */
PRB_API int prb_compute_gae(prb_ctx ctx, const float* d_rewards, const float* d_values, const uint8_t* d_dones,
                            const float* d_bootstrap, size_t num_envs, size_t horizon, double gamma, double lambda,
                            float* d_adv, float* d_ret);

/* ---- PPO (ppo.hpp:18-296) ------------------------------------------------ */
typedef struct {
  double gamma, gae_lambda, clip_eps, entropy_coef, value_coef; /* PpoConfig ppo.hpp:18-27 */
  uint64_t epochs_per_update, minibatch_size, buffer_size;
  double learning_rate;
} prb_ppo_config;

typedef struct {
  double mean_policy_loss, mean_value_loss, mean_entropy; /* PpoUpdateStats ppo.hpp:198-203 */
  uint64_t minibatches;
} prb_ppo_stats;

/* ppo_update ppo.hpp:249-296: dst := src, then epochs x full minibatches of
 * (gather, actor/critic forward, clipped surrogate + value + entropy
 * gradients, Adam).  GAE is (re)computed from r.  Permutations: if perm is
 * NULL they are generated on device from seed; else perm holds
 * epochs*buffer_size indices in the reference index space (e.g. the exact
 * std::shuffle sequence).  On error dst is unspecified and src untouched;
 * src == dst is allowed (the agent is restored on error). */
PRB_API int prb_ppo_update(prb_agent src, prb_rollout r, const prb_ppo_config* cfg, uint64_t seed,
                           const uint64_t* perm, prb_agent dst, prb_ppo_stats* stats);
/* Which device path prb_ppo_update runs when `a` is its src: 0 (default) = the
 * fp32 SIMT update over the whole GPU (reference-precision gradients, any
 * shape; the lowest latency for ONE learner); 1 = the tensor-core update
 * (ppo_tc.cu: 8 co-resident CTAs per learner, bf16 operands /
 * fp32 accumulation, for actor S-64-64-A / critic S-64-64-1 nets with A <= 32
 * and minibatches <= 1,024 rows; other shapes fall back to 0) -- the path
 * prb_ppo_update_learners always takes, where many learners share the GPU. */
PRB_API int prb_agent_set_ppo_mode(prb_agent a, int mode);
/* pod_train's learner phase (pod.hpp:436-461): L learners, learner l running
 * ppo_update(srcs[l], rollouts[l], cfg, seeds[l]) into dsts[l] -- all of them in
 * ONE cooperative launch of the tensor-core update (ceil(minibatch / 128)
 * co-resident CTAs per learner, ppo_tc.cu; 18 learners of 8 CTAs per wave on a
 * B200), so the learners of every pod on the GPU train concurrently.  Learners of one pod pass the same rollout
 * (its GAE runs once); every rollout must have the same shape.  Agents of other
 * shapes than prb_agent_set_ppo_mode lists run their updates one after another on
 * the SIMT path (same results as prb_ppo_update each).  Permutations are
 * drawn on the device from seeds[l].  stats (nullable) receives L entries.
 * NumericError if a learner's gate failed (its dst holds its last accepted
 * step; the other learners finish their updates). */
PRB_API int prb_ppo_update_learners(const prb_agent* srcs, const prb_rollout* rollouts, size_t L,
                                    const prb_ppo_config* cfg, const uint64_t* seeds, const prb_agent* dsts,
                                    prb_ppo_stats* stats);
/* detail::ppo_loss_grads ppo.hpp:116-188 on one minibatch of rollout rows
 * (reference index space); grads [P] (flat layout) and losses[3] to host.
 * Requires prb_gae first. */
PRB_API int prb_ppo_loss_grads(prb_agent a, prb_rollout r, const uint64_t* rows, size_t n, const prb_ppo_config* cfg,
                               double* grads, double* losses);
/* adam_step nn.hpp:164-182 with host gradients (NumericError, state untouched,
 * on a non-finite gradient). */
PRB_API int prb_adam_step_host(prb_agent a, const double* grads);
/* adam_step nn.hpp:164-182 with DEVICE fp32 gradients [P] (flat layout): a grid-wide
 * finite check first (NumericError, state untouched, on a non-finite gradient), then
 * the update; t advances by one on success. */
PRB_API int prb_adam_step_device(prb_agent a, const float* d_grads);

/* ---- evaluator (evaluate pod.hpp:43-83, PodEvaluator::process :313-316) --
 * `episodes` = env's num_envs evaluation episodes of the agent's policy:
 * the VecEnv is reset with the per-episode streams derive_seed(seed,
 * kEpisode, i) (its state is consumed) and stepped with the policy mean
 * clipped to the spec bounds (sample_actions != 0: Gaussian samples with
 * Philox noise in place of the reference's mt19937_64 normals).  Outputs the
 * fp64 total reward of each episode (its first done), their mean and
 * population standard deviation (EvaluationRecord), and the evaluation env
 * steps taken.  UsageError if an episode does not end within the env's step
 * bound. */
PRB_API int prb_evaluate(prb_agent a, prb_vecenv env, uint64_t seed, int sample_actions, double* episodic_rewards,
                         double* mean, double* std_dev, uint64_t* eval_steps);
/* prb_evaluate for the P pods of a GPU in one pass (one policy launch per step for every pod):
 * pod p's results equal prb_evaluate(agents[p], envs[p], seeds[p], sample_actions, ...) exactly.
 * Every eval VecEnv: the same num_envs, action dim, episode bound and context.  episodic_rewards
 * [P][num_envs]; means, std_devs, eval_steps [P] (nullable).                       pod.hpp:43-83 */
PRB_API int prb_evaluate_pods(const prb_agent* agents, const prb_vecenv* envs, size_t P, const uint64_t* seeds,
                              int sample_actions, double* episodic_rewards, double* means, double* std_devs,
                              uint64_t* eval_steps);

/* ---- learner fusion (pod.hpp:141-172) ----------------------------------- */
PRB_API int prb_fuse_parameters(const prb_agent* agents, size_t n, prb_agent out);

/* ---- leaderboard (tournament.hpp:44-162) --------------------------------- */
/* Ranks candidates (score, seq) by (score desc, seq asc) and keeps the top
 * `capacity` -- identical to sequential leaderboard_update insertion
 * (tournament.hpp:104-119).  d_order[capacity] receives candidate indices,
 * d_count the board size.  NumericError on a non-finite score. */
PRB_API int prb_leaderboard_rank(prb_ctx ctx, const double* d_scores, const uint64_t* d_seqs, size_t n,
                                 size_t capacity, int32_t* d_order, int32_t* d_count);
PRB_API int prb_leaderboard_rank_host(prb_ctx ctx, const double* scores, const uint64_t* seqs, size_t n,
                                      size_t capacity, int32_t* order, int32_t* count);
/* Leaderboard::refresh_stats tournament.hpp:66-87 (PopulationStats :38-41):
 * per-coordinate mean and population variance (divide by n) of the flat
 * parameters of the board's entries, entries[0..n) in board order, fp64 in
 * the reference's summation order.  d_mean / d_variance: [P] fp64 device
 * arrays on the entries' device.  n == 0 (empty board) writes nothing. */
PRB_API int prb_leaderboard_stats(const prb_agent* entries, size_t n, double* d_mean, double* d_variance);
PRB_API int prb_leaderboard_stats_host(const prb_agent* entries, size_t n, double* mean, double* variance);
/* generate_pod_init's mutation (tournament.hpp:149-159): params += N(0, sigma^2)
 * from a Philox stream keyed by mutation_seed; optimiser t := 0, m/v kept. */
PRB_API int prb_agent_mutate(prb_agent a, uint64_t mutation_seed, double sigma);

/* ---- checkpoints: PODRCKPT v1 (checkpoint.hpp:16-317) ---------------------
 * The byte format of encode_checkpoint(artifact_to_tensors(a, meta)): magic,
 * version 1, the named f64 tensor table (actor/critic layers, log_std, Adam
 * m / v / scalars, lineage, algo_tag, optional meta), CRC-32 (IEEE).  Readers
 * check the CRC first (CorruptionError), then magic (FormatError) and version
 * (VersionError), as the reference does.  algo_tag NULL = "ppo"; meta (nullable)
 * = (wall_seconds, env_steps, score).  With out == NULL *size receives the
 * byte count.  Decoding into an agent of other shapes is a DimensionError. */
PRB_API int prb_checkpoint_encode(prb_agent a, int64_t parent_pod, uint64_t mutation_seed, const char* algo_tag,
                                  const double* meta, uint8_t* out, size_t capacity, size_t* size);
PRB_API int prb_checkpoint_decode(prb_agent a, const uint8_t* bytes, size_t size, int64_t* parent_pod,
                                  uint64_t* mutation_seed, char* algo_tag, size_t tag_capacity, double* meta,
                                  int* has_meta);
PRB_API int prb_checkpoint_save(prb_agent a, const char* path, int64_t parent_pod, uint64_t mutation_seed,
                                const char* algo_tag, const double* meta);              /* checkpoint.hpp:305 */
PRB_API int prb_checkpoint_load(prb_agent a, const char* path, int64_t* parent_pod, uint64_t* mutation_seed,
                                char* algo_tag, size_t tag_capacity, double* meta, int* has_meta); /* :314 */
/* The same over host arrays in the flat layout (no device): hyper = (beta1,
 * beta2, eps, lr); the network is actor S-hidden-A / critic S-hidden-1. */
PRB_API int prb_checkpoint_encode_host(size_t S, size_t A, const size_t* hidden, int nh, const double* flat,
                                       const double* m, const double* v, int64_t t, const double* hyper,
                                       int64_t parent_pod, uint64_t mutation_seed, const char* algo_tag,
                                       const double* meta, uint8_t* out, size_t capacity, size_t* size);
PRB_API int prb_checkpoint_decode_host(const uint8_t* bytes, size_t size, size_t S, size_t A, const size_t* hidden,
                                       int nh, double* flat, double* m, double* v, int64_t* t, double* hyper,
                                       int64_t* parent_pod, uint64_t* mutation_seed, char* algo_tag,
                                       size_t tag_capacity, double* meta, int* has_meta);

/* ---- NCCL over NVLink (tournament C4) --------------------- */
typedef struct prb_comm_s* prb_comm;
PRB_API int prb_comm_unique_id(uint8_t id[128]);
PRB_API int prb_comm_init(prb_ctx ctx, const uint8_t id[128], int nranks, int rank, prb_comm* out);
PRB_API int prb_comm_destroy(prb_comm c);
/* All-gather of every rank's n_local (score, seq, pod_id) then the same
 * ranking on every rank.  Outputs (device): d_all_* [nranks*n_local],
 * d_order [capacity], d_count. */
PRB_API int prb_leaderboard_allgather_rank(prb_comm c, const double* d_scores, const uint64_t* d_seqs,
                                           const int64_t* d_ids, size_t n_local, size_t capacity, double* d_all_scores,
                                           uint64_t* d_all_seqs, int64_t* d_all_ids, int32_t* d_order,
                                           int32_t* d_count);
/* Broadcast an agent's params, m, v and t from `root` (elite broadcast). */
PRB_API int prb_agent_broadcast(prb_comm c, prb_agent a, int root);

/* ---- test-only switches (no reference analogue) -------------------------- */
/* Process-wide; they select alternate device paths so tests can check them
 * against the default path.  Production code never sets them. */
#define PRB_OPT_PPO_PER_KERNEL 1 /* prb_ppo_update: per-kernel path (4 launches per minibatch) */
#define PRB_OPT_TC_FORCE_REDO 2  /* stock tcgen05 rollout: exact-division redo of every step's trades */
#define PRB_OPT_PM_CTA_PAIR 3    /* PointMass 3x256 rollout: the cta_group::2 CTA-pair kernel */
PRB_API int prb_debug_set_option(int option, int value);

/* ---- self-test of the tcgen05 building block (tests only) --------------- */
/* D[128][N] = bf16(A[128][K]) . bf16(B[N][K])^T with fp32 accumulation in
 * TMEM, one CTA, K % 16 == 0 (<= 256), N % 16 == 0 (<= 256). */
PRB_API int prb_debug_tc_gemm(prb_ctx ctx, int K, int N, const float* A, const float* B, float* D);

/* The same GEMM with A and/or B stored transposed (MN-major operands, the
 * layout the PPO backward uses); hyp selects the descriptor stride convention
 * under test (0: LBO along MN, SBO along K; 1: swapped). */
PRB_API int prb_debug_tc_gemm_major(prb_ctx ctx, int K, int N, int a_mn, int b_mn, int hyp, const float* A,
                                    const float* B, float* D);

/* The reduced gradient [P] (flat layout) of the last minibatch step the
 * tensor-core PPO update ran on `a` (its dst), or of the last
 * prb_adam_step_device / per-kernel step (tests only). */
PRB_API int prb_debug_agent_grads(prb_agent a, double* grads);

/* ---- self-test of the fused rollout's trade arithmetic (tests only) ------ */
/* Per element i, the device functions the tcgen05 stock rollout uses for
 * stock_env_step (stock_env.hpp:83-97): desired[i] = trunc(clamp(act[i],-1,1)
 * * max_trade) and buy[i] = buy_i[i] = min(desired, max(floor(balance /
 * (price * (1 + cost_rate))), 0)) (for desired > 0; desired <= 0 is no buy in the
 * reference and gives 0).  max_trade: integer < 2^22. */
PRB_API int prb_debug_trade_math(prb_ctx ctx, size_t n, const float* act, double max_trade, const double* balance,
                                 const double* price, double cost_rate, int32_t* desired, double* buy,
                                 int32_t* buy_i);

#ifdef __cplusplus
}
#endif
#endif /* PRB_H_ */
