/*
 * podracer_oracle.c -- TEST INFRASTRUCTURE ONLY (the parity checker).
 *
 * A plain-C, scalar-double restatement of the reference's pod hot path
 * (ElegantRL-podracer restated in /root/reference/proj/include/podracer/*.hpp).
 * Every function cites the reference file:line it follows.  Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline leg may load this
 * library; the product path (paper_2112_05923_b200/) never links or calls it.
 *
 * Pinning: tests/test_oracle_pinned.py checks every function here against the
 * reference itself (oracle/_ref/libpodracer_ref_exact.so, built from the
 * reference headers by oracle/Makefile with the same -ffp-contract=off flags)
 * and against the known-answer tests the reference's unit tests hold.
 *
 * Build flags are part of the contract: -O2 -ffp-contract=off (no FMA
 * contraction), so floating-point results are a pure function of the IEEE
 * operation order written here.
 *
 * Layouts (all row-major, matching the reference):
 *   MLP layer i: W [dims[i] x dims[i+1]] then b [dims[i+1]]   (nn.hpp:16-24)
 *   agent flat:  actor layers, log_std[A], critic layers       (artifact.hpp:35-51)
 *   market:      close[k*T + t], indicators[(i*K + k)*T + t]  (market.hpp:104-113)
 */
#include <math.h>
#include <stddef.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORC_API __attribute__((visibility("default")))

static const double kLogTwoPi = 1.8378770664093454836; /* nn.hpp:209 */

/* ------------------------------------------------------------------------- */
/* Seeds: common.hpp:79-93                                                    */
/* ------------------------------------------------------------------------- */

ORC_API uint64_t orc_splitmix64(uint64_t x) { /* common.hpp:79-84 */
  x += 0x9e3779b97f4a7c15ULL;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}

/* derive_seed(base, tags...) : common.hpp:88-93 */
ORC_API uint64_t orc_derive_seed(uint64_t base, const uint64_t* tags, int ntags) {
  uint64_t s = orc_splitmix64(base);
  for (int i = 0; i < ntags; ++i) s = orc_splitmix64(s ^ orc_splitmix64(tags[i]));
  return s;
}

/* ------------------------------------------------------------------------- */
/* mt19937_64 + libstdc++ uniform_real_distribution<double>: the per-env reset */
/* stream of VectorizedEnvironment::reset (env.hpp:186-194) and PointMass2D    */
/* ::reset (env.hpp:124-133).  Published algorithm (C++11 [rand.predef],       */
/* Matsumoto & Nishimura); canonical mapping as libstdc++ 13                   */
/* bits/random.tcc generate_canonical<double,53>: u = double(x) / 2^64.        */
/* ------------------------------------------------------------------------- */

typedef struct {
  uint64_t mt[312];
  int idx;
} orc_mt64;

ORC_API void orc_mt64_seed(orc_mt64* g, uint64_t seed) {
  g->mt[0] = seed;
  for (int i = 1; i < 312; ++i)
    g->mt[i] = 6364136223846793005ULL * (g->mt[i - 1] ^ (g->mt[i - 1] >> 62)) + (uint64_t)i;
  g->idx = 312;
}

ORC_API uint64_t orc_mt64_next(orc_mt64* g) {
  if (g->idx >= 312) {
    const uint64_t upper = 0xFFFFFFFF80000000ULL, lower = 0x7FFFFFFFULL;
    for (int i = 0; i < 312; ++i) {
      uint64_t y = (g->mt[i] & upper) | (g->mt[(i + 1) % 312] & lower);
      uint64_t v = g->mt[(i + 156) % 312] ^ (y >> 1);
      if (y & 1ULL) v ^= 0xB5026F5AA96619E9ULL;
      g->mt[i] = v;
    }
    g->idx = 0;
  }
  uint64_t x = g->mt[g->idx++];
  x ^= (x >> 29) & 0x5555555555555555ULL;
  x ^= (x << 17) & 0x71D67FFFEDA60000ULL;
  x ^= (x << 37) & 0xFFF7EEE000000000ULL;
  x ^= (x >> 43);
  return x;
}

ORC_API double orc_mt64_canonical(orc_mt64* g) {
  double r = (double)orc_mt64_next(g) / 18446744073709551616.0;
  if (r >= 1.0) r = nextafter(1.0, 0.0);
  return r;
}

ORC_API double orc_uniform_real(orc_mt64* g, double a, double b) {
  const double u = orc_mt64_canonical(g);
  return u * (b - a) + a; /* no contraction: mul then add */
}

/* ------------------------------------------------------------------------- */
/* Philox4x32-10 (Salmon et al., SC'11).  Not in the reference: it is the      */
/* device's counter-based stream for policy noise, restated here so the       */
/* checker can regenerate the exact draws the GPU used.                       */
/* ------------------------------------------------------------------------- */

ORC_API void orc_philox4x32_10(uint32_t key0, uint32_t key1, const uint32_t ctr_in[4], uint32_t out[4]) {
  uint32_t c0 = ctr_in[0], c1 = ctr_in[1], c2 = ctr_in[2], c3 = ctr_in[3];
  uint32_t k0 = key0, k1 = key1;
  for (int r = 0; r < 10; ++r) {
    uint64_t p0 = (uint64_t)0xD2511F53u * c0;
    uint64_t p1 = (uint64_t)0xCD9E8D57u * c2;
    uint32_t n0 = (uint32_t)(p1 >> 32) ^ c1 ^ k0;
    uint32_t n1 = (uint32_t)p1;
    uint32_t n2 = (uint32_t)(p0 >> 32) ^ c3 ^ k1;
    uint32_t n3 = (uint32_t)p0;
    c0 = n0; c1 = n1; c2 = n2; c3 = n3;
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
  out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

/* ------------------------------------------------------------------------- */
/* Stock-trading env: stock_env.hpp:55-131, StockTradingEnv stock_env.hpp:135-184 */
/* ------------------------------------------------------------------------- */

typedef struct {
  double initial_capital;  /* stock_env.hpp:16 */
  double max_trade_shares; /* stock_env.hpp:17 */
  double cost_rate;        /* stock_env.hpp:18 */
} orc_stock_cfg;

static double clampd(double x, double lo, double hi) { return x < lo ? lo : (hi < x ? hi : x); }
static double mind(double a, double b) { return (b < a) ? b : a; } /* std::min */
static double maxd(double a, double b) { return (a < b) ? b : a; } /* std::max */

/* PortfolioState::account_value, stock_env.hpp:27-31 */
static double account_value(double balance, const double* shares, const double* close, size_t T, int K,
                            size_t t) {
  double v = balance;
  for (int k = 0; k < K; ++k) v += shares[k] * close[(size_t)k * T + t];
  return v;
}

/* stock_env_step, stock_env.hpp:55-103.  Returns 0, or 3 (UsageError) when t+1 >= T. */
ORC_API int orc_stock_env_step(double* balance, double* shares, size_t* t, const double* action,
                               const double* close, size_t T, int K, const orc_stock_cfg* cfg,
                               double* reward, int* done) {
  const size_t t0 = *t;
  if (t0 + 1 >= T) return 3; /* :64-66 */
  const double value_before = account_value(*balance, shares, close, T, K, t0); /* :68 */
  double desired[512];
  for (int k = 0; k < K; ++k) { /* :83-87 */
    const double a = clampd(action[k], -1.0, 1.0);
    desired[k] = trunc(a * cfg->max_trade_shares);
  }
#define ORC_EXECUTE(k, qty)                                                                \
  do {                                                                                     \
    const double price_ = close[(size_t)(k) * T + t0];                                     \
    const double cost_ = cfg->cost_rate * fabs(qty) * price_;                              \
    *balance -= (qty) * price_ + cost_;                                                    \
    shares[k] += (qty);                                                                    \
  } while (0) /* execute, :72-81 */
  for (int k = 0; k < K; ++k) { /* sells first, :88-90 */
    if (desired[k] < 0.0) {
      const double q = -mind(-desired[k], shares[k]);
      ORC_EXECUTE(k, q);
    }
  }
  for (int k = 0; k < K; ++k) { /* then buys, :91-97 */
    if (desired[k] > 0.0) {
      const double price = close[(size_t)k * T + t0];
      const double affordable = floor(*balance / (price * (1.0 + cfg->cost_rate)));
      const double q = mind(desired[k], maxd(affordable, 0.0));
      ORC_EXECUTE(k, q);
    }
  }
#undef ORC_EXECUTE
  *t = t0 + 1; /* :99 */
  *reward = account_value(*balance, shares, close, T, K, *t) - value_before; /* :100 */
  *done = (*t + 1 >= T); /* :101 */
  return 0;
}

/* stock_observation, stock_env.hpp:111-131 (state_dim = 1 + 6K) */
ORC_API void orc_stock_observation(double balance, const double* shares, size_t t, const double* close,
                                   const double* indicators, size_t T, int K, const orc_stock_cfg* cfg,
                                   size_t window_start, double* obs) {
  size_t j = 0;
  obs[j++] = balance / cfg->initial_capital;
  for (int k = 0; k < K; ++k) obs[j++] = shares[k];
  for (int k = 0; k < K; ++k) obs[j++] = close[(size_t)k * T + t] / close[(size_t)k * T + window_start];
  for (int i = 0; i < 4; ++i)
    for (int k = 0; k < K; ++k) obs[j++] = indicators[((size_t)i * K + k) * T + t];
}

/* VectorizedEnvironment over StockTradingEnv: reset env.hpp:186-194 +
 * stock_env.hpp:158-163, step env.hpp:200-236 + stock_env.hpp:165-170.
 * State arrays: balance[N], shares[N*K], t[N], step_count[N], ep_return[N]. */
ORC_API void orc_stock_vec_reset(size_t N, int K, const orc_stock_cfg* cfg, size_t start, double* balance,
                                 double* shares, size_t* t, size_t* step_count, double* ep_return) {
  for (size_t e = 0; e < N; ++e) {
    balance[e] = cfg->initial_capital;
    for (int k = 0; k < K; ++k) shares[e * K + k] = 0.0;
    t[e] = start;
    step_count[e] = 0;
    ep_return[e] = 0.0;
  }
}

/* One VecEnv step.  actions [N*K] (double, unclipped).  Outputs: next_obs
 * [N*S] (post auto-reset), reward[N], done[N], terminal_obs[N*S] (rows with
 * done only), term_return[N], term_len[N].  Returns 0 or 3 (UsageError). */
ORC_API int orc_stock_vec_step(size_t N, int K, const orc_stock_cfg* cfg, size_t start, size_t end,
                               const double* close, const double* indicators, size_t T, double* balance,
                               double* shares, size_t* t, size_t* step_count, double* ep_return,
                               const double* actions, double* next_obs, double* reward, uint8_t* done,
                               double* terminal_obs, double* term_return, uint64_t* term_len) {
  const size_t S = 1 + 6 * (size_t)K;
  double clipped[512];
  for (size_t e = 0; e < N; ++e) {
    for (int k = 0; k < K; ++k) clipped[k] = clampd(actions[e * K + k], -1.0, 1.0); /* env.hpp:213-215 */
    double r;
    int d;
    int rc = orc_stock_env_step(&balance[e], &shares[e * K], &t[e], clipped, close, T, K, cfg, &r, &d);
    if (rc) return rc;
    d = d || (t[e] >= end); /* stock_env.hpp:168 */
    step_count[e] += 1;     /* env.hpp:217-218 */
    ep_return[e] += r;
    reward[e] = r;
    done[e] = d ? 1 : 0;
    double* row = next_obs + e * S;
    orc_stock_observation(balance[e], &shares[e * K], t[e], close, indicators, T, K, cfg, start, row);
    if (d) { /* env.hpp:221-229 */
      memcpy(terminal_obs + e * S, row, S * sizeof(double));
      term_return[e] = ep_return[e];
      term_len[e] = step_count[e];
      balance[e] = cfg->initial_capital;
      for (int k = 0; k < K; ++k) shares[e * K + k] = 0.0;
      t[e] = start;
      orc_stock_observation(balance[e], &shares[e * K], t[e], close, indicators, T, K, cfg, start, row);
      step_count[e] = 0;
      ep_return[e] = 0.0;
    }
  }
  return 0;
}

/* ------------------------------------------------------------------------- */
/* PointMass2D: pointmass_step env.hpp:84-109, reset env.hpp:124-133          */
/* ------------------------------------------------------------------------- */

ORC_API void orc_pointmass_step(const double* s, const double* a, uint64_t steps_taken, double* out,
                                double* reward, int* done) {
  double action_sq = 0.0;
  for (int d = 0; d < 2; ++d) { /* :91-97 */
    const double vel = 0.9 * s[2 + d] + 0.1 * a[d];
    out[2 + d] = vel;
    out[d] = s[d] + 0.1 * vel;
    out[4 + d] = s[4 + d];
    action_sq += a[d] * a[d];
  }
  const double dx = out[0] - out[4];
  const double dy = out[1] - out[5];
  const double dist = sqrt(dx * dx + dy * dy); /* :100 */
  double r = -dist - 0.01 * action_sq;
  const int reached = dist < 0.05;
  if (reached) r += 10.0;
  *reward = r;
  *done = reached || (steps_taken + 1 >= 200); /* :106 */
}

/* PointMass2D::reset with the env's own stream (env.hpp:124-133). */
ORC_API void orc_pointmass_reset(orc_mt64* g, double* s) {
  s[0] = orc_uniform_real(g, -0.4, 0.4);
  s[1] = orc_uniform_real(g, -0.4, 0.4);
  s[2] = 0.0;
  s[3] = 0.0;
  s[4] = orc_uniform_real(g, -0.4, 0.4);
  s[5] = orc_uniform_real(g, -0.4, 0.4);
}

/* VectorizedEnvironment<PointMass2D>::reset(seed): env.hpp:186-194.
 * gens[N] are (re)seeded with derive_seed(seed, kVecEnv, i). */
ORC_API void orc_pm_vec_reset(size_t N, uint64_t seed, orc_mt64* gens, double* state, uint64_t* step_count,
                              double* ep_return) {
  for (size_t e = 0; e < N; ++e) {
    uint64_t tags[2] = {1 /* kVecEnv */, (uint64_t)e};
    orc_mt64_seed(&gens[e], orc_derive_seed(seed, tags, 2));
    orc_pointmass_reset(&gens[e], state + e * 6);
    step_count[e] = 0;
    ep_return[e] = 0.0;
  }
}

/* The same reset for a subset of a VecEnv's envs: env idx[i]'s generator and state land in slot
 * i (each env's stream depends only on its own index, env.hpp:186-194), so a sample of a large
 * VecEnv replays without materialising every env. */
ORC_API void orc_pm_vec_reset_subset(size_t n, const uint64_t* idx, uint64_t seed, orc_mt64* gens, double* state,
                                     uint64_t* step_count, double* ep_return) {
  for (size_t i = 0; i < n; ++i) {
    uint64_t tags[2] = {1 /* kVecEnv */, idx[i]};
    orc_mt64_seed(&gens[i], orc_derive_seed(seed, tags, 2));
    orc_pointmass_reset(&gens[i], state + i * 6);
    step_count[i] = 0;
    ep_return[i] = 0.0;
  }
}

/* VectorizedEnvironment<PointMass2D>::step: env.hpp:200-236. */
ORC_API void orc_pm_vec_step(size_t N, orc_mt64* gens, double* state, uint64_t* step_count, double* ep_return,
                             const double* actions, double* reward, uint8_t* done, double* terminal_state,
                             double* term_return, uint64_t* term_len) {
  for (size_t e = 0; e < N; ++e) {
    double a[2], nxt[6], r;
    int d;
    a[0] = clampd(actions[e * 2 + 0], -1.0, 1.0);
    a[1] = clampd(actions[e * 2 + 1], -1.0, 1.0);
    orc_pointmass_step(state + e * 6, a, step_count[e], nxt, &r, &d);
    step_count[e] += 1;
    ep_return[e] += r;
    reward[e] = r;
    done[e] = d ? 1 : 0;
    if (d) {
      memcpy(terminal_state + e * 6, nxt, sizeof nxt);
      term_return[e] = ep_return[e];
      term_len[e] = step_count[e];
      orc_pointmass_reset(&gens[e], state + e * 6);
      step_count[e] = 0;
      ep_return[e] = 0.0;
    } else {
      memcpy(state + e * 6, nxt, sizeof nxt);
    }
  }
}

/* ------------------------------------------------------------------------- */
/* MLP: mlp_forward nn.hpp:63-85 (matmul tensor.hpp:43-81, add_row_vector     */
/* tensor.hpp:163-172), tanh hidden / linear output.                           */
/* ------------------------------------------------------------------------- */

static size_t mlp_param_count(const size_t* dims, int nlayers) {
  size_t n = 0;
  for (int i = 0; i < nlayers; ++i) n += dims[i] * dims[i + 1] + dims[i + 1];
  return n;
}

ORC_API size_t orc_mlp_param_count(const size_t* dims, int nlayers) { return mlp_param_count(dims, nlayers); }

/* acts (optional): concatenation of post-activation outputs of every layer,
 * layer i occupying n*dims[i+1] doubles (MlpCache::acts[1..], nn.hpp:58-61). */
ORC_API void orc_mlp_forward(const double* params, const size_t* dims, int nlayers, const double* X, size_t n,
                             double* Y, double* acts) {
  size_t maxw = 0;
  for (int i = 0; i <= nlayers; ++i) maxw = dims[i] > maxw ? dims[i] : maxw;
  double* h = (double*)malloc(sizeof(double) * n * maxw);
  double* z = (double*)malloc(sizeof(double) * n * maxw);
  memcpy(h, X, sizeof(double) * n * dims[0]);
  const double* p = params;
  size_t act_off = 0;
  for (int li = 0; li < nlayers; ++li) {
    const size_t in = dims[li], out = dims[li + 1];
    const double* W = p;
    const double* b = p + in * out;
    for (size_t i = 0; i < n; ++i) {
      for (size_t j = 0; j < out; ++j) z[i * out + j] = 0.0;
      for (size_t k = 0; k < in; ++k) {
        const double a = h[i * in + k];
        for (size_t j = 0; j < out; ++j) z[i * out + j] += a * W[k * out + j];
      }
      for (size_t j = 0; j < out; ++j) z[i * out + j] += b[j];
      if (li + 1 < nlayers)
        for (size_t j = 0; j < out; ++j) z[i * out + j] = tanh(z[i * out + j]);
    }
    if (acts) {
      memcpy(acts + act_off, z, sizeof(double) * n * out);
      act_off += n * out;
    }
    memcpy(h, z, sizeof(double) * n * out);
    p += in * out + out;
  }
  memcpy(Y, h, sizeof(double) * n * dims[nlayers]);
  free(h);
  free(z);
}

/* detail::gaussian_row_log_prob, nn.hpp:215-224 */
ORC_API double orc_gaussian_row_log_prob(const double* log_std, int A, const double* mean_row,
                                         const double* action_row) {
  double acc = 0.0;
  for (int d = 0; d < A; ++d) {
    const double sigma = exp(log_std[d]);
    const double z = (action_row[d] - mean_row[d]) / sigma;
    acc += -0.5 * kLogTwoPi - log_std[d] - 0.5 * z * z;
  }
  return acc;
}

/* policy_sample nn.hpp:250-265 with the unit-normal draws injected (the device
 * draws them from Philox; std::normal_distribution is not reproducible). */
ORC_API void orc_policy_sample_eps(const double* actor_params, const size_t* dims, int nlayers,
                                   const double* log_std, const double* states, size_t n, const double* eps,
                                   double* actions, double* log_probs) {
  const int A = (int)dims[nlayers];
  double* mean = (double*)malloc(sizeof(double) * n * A);
  orc_mlp_forward(actor_params, dims, nlayers, states, n, mean, NULL);
  for (size_t i = 0; i < n; ++i) {
    for (int d = 0; d < A; ++d) actions[i * A + d] = mean[i * A + d] + exp(log_std[d]) * eps[i * A + d];
    log_probs[i] = orc_gaussian_row_log_prob(log_std, A, mean + i * A, actions + i * A);
  }
  free(mean);
}

/* policy_entropy nn.hpp:273-277 */
ORC_API double orc_policy_entropy(const double* log_std, int A) {
  double h = 0.0;
  for (int d = 0; d < A; ++d) h += 0.5 * (kLogTwoPi + 1.0) + log_std[d];
  return h;
}

/* ------------------------------------------------------------------------- */
/* GAE: compute_gae ppo.hpp:50-71; buffer_advantages ppo.hpp:212-244          */
/* ------------------------------------------------------------------------- */

ORC_API void orc_compute_gae(const double* r, const double* v, const uint8_t* d, size_t T, double bootstrap,
                             double gamma, double lambda, double* adv, double* ret) {
  double gae = 0.0;
  for (size_t i = T; i-- > 0;) {
    const double next_value = (i + 1 < T) ? v[i + 1] : bootstrap;
    const double nonterminal = d[i] ? 0.0 : 1.0;
    const double delta = r[i] + gamma * next_value * nonterminal - v[i];
    gae = delta + gamma * lambda * nonterminal * gae;
    adv[i] = gae;
    ret[i] = gae + v[i];
  }
}

/* Chunks: offsets[c], lengths[c], bootstrap[c].  Returns 3 on incomplete coverage. */
ORC_API int orc_buffer_advantages(const double* r, const double* v, const uint8_t* d, size_t n,
                                  const size_t* offsets, const size_t* lengths, const double* bootstrap,
                                  size_t nchunks, double gamma, double lambda, int normalize, double* adv,
                                  double* ret) {
  size_t covered = 0;
  for (size_t c = 0; c < nchunks; ++c) {
    orc_compute_gae(r + offsets[c], v + offsets[c], d + offsets[c], lengths[c], bootstrap[c], gamma, lambda,
                    adv + offsets[c], ret + offsets[c]);
    covered += lengths[c];
  }
  if (covered != n) return 3; /* :230-233 */
  if (normalize && n > 0) {   /* :234-242 */
    const double nn = (double)n;
    double mean = 0.0;
    for (size_t i = 0; i < n; ++i) mean += adv[i];
    mean /= nn;
    double var = 0.0;
    for (size_t i = 0; i < n; ++i) var += (adv[i] - mean) * (adv[i] - mean);
    var /= nn;
    const double denom = maxd(sqrt(var), 1e-8);
    for (size_t i = 0; i < n; ++i) adv[i] = (adv[i] - mean) / denom;
  }
  return 0;
}

/* ------------------------------------------------------------------------- */
/* Backprop: mlp_backward_accumulate nn.hpp:105-132 with the reference's      */
/* 4-row-blocked matmul_tn (tensor.hpp:85-119), matmul_nt (:122-160),          */
/* column_sums (:175-183).  grads laid out like params (accumulated).          */
/* ------------------------------------------------------------------------- */

static void mlp_backward(const double* params, const size_t* dims, int nlayers, const double* X,
                         const double* acts, size_t n, const double* upstream, double* grads) {
  size_t maxw = 0;
  for (int i = 0; i <= nlayers; ++i) maxw = dims[i] > maxw ? dims[i] : maxw;
  double* delta = (double*)malloc(sizeof(double) * n * maxw);
  double* dprev = (double*)malloc(sizeof(double) * n * maxw);
  double* dw = (double*)malloc(sizeof(double) * maxw * maxw);
  memcpy(delta, upstream, sizeof(double) * n * dims[nlayers]);
  /* offsets of each layer's params and activations */
  size_t poff[64], aoff[64];
  size_t po = 0, ao = 0;
  for (int i = 0; i < nlayers; ++i) {
    poff[i] = po;
    po += dims[i] * dims[i + 1] + dims[i + 1];
    aoff[i] = ao;
    ao += n * dims[i + 1];
  }
  for (int li = nlayers; li-- > 0;) {
    const size_t in = dims[li], out = dims[li + 1];
    const double* layer_in = (li == 0) ? X : acts + aoff[li - 1];
    /* dw = matmul_tn(layer_in, delta) */
    for (size_t i = 0; i < in * out; ++i) dw[i] = 0.0;
    size_t k = 0;
    for (; k + 4 <= n; k += 4) {
      const double *a0 = layer_in + k * in, *a1 = a0 + in, *a2 = a1 + in, *a3 = a2 + in;
      const double *b0 = delta + k * out, *b1 = b0 + out, *b2 = b1 + out, *b3 = b2 + out;
      for (size_t i = 0; i < in; ++i) {
        const double w0 = a0[i], w1 = a1[i], w2 = a2[i], w3 = a3[i];
        double* crow = dw + i * out;
        for (size_t j = 0; j < out; ++j) crow[j] += w0 * b0[j] + w1 * b1[j] + w2 * b2[j] + w3 * b3[j];
      }
    }
    for (; k < n; ++k) {
      const double* arow = layer_in + k * in;
      const double* brow = delta + k * out;
      for (size_t i = 0; i < in; ++i) {
        const double aki = arow[i];
        double* crow = dw + i * out;
        for (size_t j = 0; j < out; ++j) crow[j] += aki * brow[j];
      }
    }
    double* gW = grads + poff[li];
    double* gb = gW + in * out;
    for (size_t i = 0; i < in * out; ++i) gW[i] += dw[i];
    for (size_t j = 0; j < out; ++j) {
      double s = 0.0;
      for (size_t r = 0; r < n; ++r) s += delta[r * out + j];
      gb[j] += s;
    }
    if (li == 0) break;
    /* dprev = matmul_nt(delta, W) then * (1 - a^2) */
    const double* W = params + poff[li];
    const double* a = acts + aoff[li - 1];
    for (size_t r = 0; r < n; ++r) {
      for (size_t j = 0; j < in; ++j) {
        double dot = 0.0;
        for (size_t q = 0; q < out; ++q) dot += delta[r * out + q] * W[j * out + q];
        dprev[r * in + j] = dot;
      }
    }
    for (size_t i = 0; i < n * in; ++i) dprev[i] *= (1.0 - a[i] * a[i]);
    memcpy(delta, dprev, sizeof(double) * n * in);
  }
  free(delta);
  free(dprev);
  free(dw);
}

/* ------------------------------------------------------------------------- */
/* PPO loss + grads: detail::ppo_loss_grads ppo.hpp:116-188                   */
/* ------------------------------------------------------------------------- */

typedef struct {
  double gamma, gae_lambda, clip_eps, entropy_coef, value_coef; /* ppo.hpp:18-23 */
  uint64_t epochs_per_update, minibatch_size, buffer_size;    /* ppo.hpp:24-26 */
  double learning_rate;                                       /* ppo.hpp:27 */
} orc_ppo_cfg;

/* agent flat = [actor params | log_std | critic params] (artifact.hpp:35-51).
 * adims: actor dims (nl_a layers), cdims: critic dims (nl_c layers, last = 1).
 * mb_*: gathered minibatch rows (gather_minibatch ppo.hpp:83-103).
 * grads (optional) receives the flat gradient.  losses[3] = policy, value, entropy.
 * Returns 0, or 2 (NumericError) on a non-finite loss (ppo.hpp:169-171). */
ORC_API int orc_ppo_loss_grads(const double* flat, const size_t* adims, int nl_a, const size_t* cdims, int nl_c,
                               const double* mb_states, const double* mb_actions, const double* mb_old_lp,
                               const double* mb_adv, const double* mb_ret, size_t n, const orc_ppo_cfg* cfg,
                               double* grads, double* losses) {
  const int A = (int)adims[nl_a];
  const size_t pa = mlp_param_count(adims, nl_a);
  const size_t pc = mlp_param_count(cdims, nl_c);
  const double* actor = flat;
  const double* log_std = flat + pa;
  const double* critic = flat + pa + A;
  const double inv_n = 1.0 / (double)n;
  size_t a_acts = 0, c_acts = 0;
  for (int i = 0; i < nl_a; ++i) a_acts += n * adims[i + 1];
  for (int i = 0; i < nl_c; ++i) c_acts += n * cdims[i + 1];
  double* acts_a = (double*)malloc(sizeof(double) * a_acts);
  double* acts_c = (double*)malloc(sizeof(double) * c_acts);
  double* mean = (double*)malloc(sizeof(double) * n * A);
  double* dmean = (double*)calloc(n * A, sizeof(double));
  double* value = (double*)malloc(sizeof(double) * n);
  double* dvalue = (double*)calloc(n, sizeof(double));
  double dlog_std[512];
  for (int d = 0; d < A; ++d) dlog_std[d] = 0.0;
  orc_mlp_forward(actor, adims, nl_a, mb_states, n, mean, acts_a);
  double policy_loss = 0.0, value_loss = 0.0;
  for (size_t i = 0; i < n; ++i) { /* :128-154 */
    double lp = 0.0;
    for (int d = 0; d < A; ++d) {
      const double sigma = exp(log_std[d]);
      const double z = (mb_actions[i * A + d] - mean[i * A + d]) / sigma;
      lp += -0.5 * kLogTwoPi - log_std[d] - 0.5 * z * z;
    }
    const double ratio = exp(lp - mb_old_lp[i]);
    const double adv = mb_adv[i];
    const double surr1 = ratio * adv;
    const double clipped = clampd(ratio, 1.0 - cfg->clip_eps, 1.0 + cfg->clip_eps);
    const double surr2 = clipped * adv;
    policy_loss += -mind(surr1, surr2) * inv_n;
    if (grads) {
      const double dl_dlp = (surr1 <= surr2) ? -adv * ratio * inv_n : 0.0; /* :146 */
      for (int d = 0; d < A; ++d) {
        const double sigma = exp(log_std[d]);
        const double z = (mb_actions[i * A + d] - mean[i * A + d]) / sigma;
        dmean[i * A + d] = dl_dlp * (z / sigma);
        dlog_std[d] += dl_dlp * (z * z - 1.0);
      }
    }
  }
  const double entropy = orc_policy_entropy(log_std, A); /* :155 */
  if (grads)
    for (int d = 0; d < A; ++d) dlog_std[d] -= cfg->entropy_coef; /* :157 */
  orc_mlp_forward(critic, cdims, nl_c, mb_states, n, value, acts_c); /* :161 */
  for (size_t i = 0; i < n; ++i) {                                    /* :162-167 */
    const double err = value[i] - mb_ret[i];
    value_loss += err * err * inv_n;
    if (grads) dvalue[i] = cfg->value_coef * 2.0 * err * inv_n;
  }
  losses[0] = policy_loss;
  losses[1] = value_loss;
  losses[2] = entropy;
  int rc = 0;
  if (!isfinite(policy_loss) || !isfinite(value_loss) || !isfinite(entropy)) rc = 2;
  if (!rc && grads) { /* :173-185 */
    memset(grads, 0, sizeof(double) * (pa + A + pc));
    mlp_backward(actor, adims, nl_a, mb_states, acts_a, n, dmean, grads);
    for (int d = 0; d < A; ++d) grads[pa + d] = dlog_std[d];
    mlp_backward(critic, cdims, nl_c, mb_states, acts_c, n, dvalue, grads + pa + A);
  }
  free(acts_a);
  free(acts_c);
  free(mean);
  free(dmean);
  free(value);
  free(dvalue);
  return rc;
}

/* adam_step nn.hpp:164-182.  Returns 2 (NumericError) on non-finite grads
 * before touching any state (:169-171). */
ORC_API int orc_adam_step(double* params, const double* grads, double* m, double* v, int64_t* t, size_t n,
                          double beta1, double beta2, double eps, double lr) {
  for (size_t i = 0; i < n; ++i)
    if (!isfinite(grads[i])) return 2;
  *t += 1;
  const double bc1 = 1.0 - pow(beta1, (double)*t);
  const double bc2 = 1.0 - pow(beta2, (double)*t);
  for (size_t i = 0; i < n; ++i) {
    m[i] = beta1 * m[i] + (1.0 - beta1) * grads[i];
    v[i] = beta2 * v[i] + (1.0 - beta2) * grads[i] * grads[i];
    const double mhat = m[i] / bc1;
    const double vhat = v[i] / bc2;
    params[i] -= lr * mhat / (sqrt(vhat) + eps);
  }
  return 0;
}

/* ppo_update ppo.hpp:249-296 with the per-epoch permutations injected
 * (perms[epoch*n + j]); the reference draws them with std::shuffle.
 * Buffer arrays are in the reference's index space; chunks as in
 * orc_buffer_advantages.  Updates flat/m/v/t in place; stats[4] = mean
 * policy, value, entropy losses and the minibatch count. */
ORC_API int orc_ppo_update(double* flat, double* m, double* v, int64_t* t, const size_t* adims, int nl_a,
                           const size_t* cdims, int nl_c, const double* states, const double* actions,
                           const double* log_probs, const double* rewards, const uint8_t* dones,
                           const double* values, size_t n, int S, const size_t* offsets, const size_t* lengths,
                           const double* bootstrap, size_t nchunks, const orc_ppo_cfg* cfg, const uint64_t* perms,
                           double* stats) {
  const int A = (int)adims[nl_a];
  const size_t P = mlp_param_count(adims, nl_a) + (size_t)A + mlp_param_count(cdims, nl_c);
  double* adv = (double*)malloc(sizeof(double) * n);
  double* ret = (double*)malloc(sizeof(double) * n);
  int rc = orc_buffer_advantages(rewards, values, dones, n, offsets, lengths, bootstrap, nchunks, cfg->gamma,
                                 cfg->gae_lambda, 1, adv, ret);
  const size_t mb = cfg->minibatch_size;
  double* ms = (double*)malloc(sizeof(double) * mb * S);
  double* ma = (double*)malloc(sizeof(double) * mb * A);
  double* mlp = (double*)malloc(sizeof(double) * mb);
  double* madv = (double*)malloc(sizeof(double) * mb);
  double* mret = (double*)malloc(sizeof(double) * mb);
  double* grads = (double*)malloc(sizeof(double) * P);
  double losses[3];
  stats[0] = stats[1] = stats[2] = stats[3] = 0.0;
  for (uint64_t ep = 0; !rc && ep < cfg->epochs_per_update; ++ep) {
    const uint64_t* idx = perms + ep * n;
    for (size_t start = 0; !rc && start + mb <= n; start += mb) {
      for (size_t r = 0; r < mb; ++r) { /* gather_minibatch ppo.hpp:83-103 */
        const size_t i = (size_t)idx[start + r];
        memcpy(ms + r * S, states + i * S, sizeof(double) * S);
        memcpy(ma + r * A, actions + i * A, sizeof(double) * A);
        mlp[r] = log_probs[i];
        madv[r] = adv[i];
        mret[r] = ret[i];
      }
      rc = orc_ppo_loss_grads(flat, adims, nl_a, cdims, nl_c, ms, ma, mlp, madv, mret, mb, cfg, grads, losses);
      if (rc) break;
      rc = orc_adam_step(flat, grads, m, v, t, P, 0.9, 0.999, 1e-8, cfg->learning_rate);
      stats[0] += losses[0];
      stats[1] += losses[1];
      stats[2] += losses[2];
      stats[3] += 1.0;
    }
  }
  if (stats[3] > 0) {
    stats[0] /= stats[3];
    stats[1] /= stats[3];
    stats[2] /= stats[3];
  }
  free(adv); free(ret); free(ms); free(ma); free(mlp); free(madv); free(mret); free(grads);
  return rc;
}

/* ------------------------------------------------------------------------- */
/* fuse_parameters pod.hpp:141-172 over L flat blobs (params, m, v, t)        */
/* ------------------------------------------------------------------------- */

ORC_API void orc_fuse(const double* const* params, const double* const* m, const double* const* v,
                      const int64_t* t, size_t L, size_t P, double* out_p, double* out_m, double* out_v,
                      int64_t* out_t) {
  if (L == 1) {
    memcpy(out_p, params[0], sizeof(double) * P);
    memcpy(out_m, m[0], sizeof(double) * P);
    memcpy(out_v, v[0], sizeof(double) * P);
    *out_t = t[0];
    return;
  }
  const double inv = 1.0 / (double)L;
  for (size_t i = 0; i < P; ++i) out_p[i] = out_m[i] = out_v[i] = 0.0;
  int64_t tt = 0;
  for (size_t a = 0; a < L; ++a) {
    for (size_t i = 0; i < P; ++i) out_p[i] += params[a][i];
    for (size_t i = 0; i < P; ++i) {
      out_m[i] += m[a][i];
      out_v[i] += v[a][i];
    }
    tt = t[a] > tt ? t[a] : tt;
  }
  for (size_t i = 0; i < P; ++i) {
    out_p[i] *= inv;
    out_m[i] *= inv;
    out_v[i] *= inv;
  }
  *out_t = tt;
}

/* ------------------------------------------------------------------------- */
/* Leaderboard: leaderboard_update tournament.hpp:104-119 on (score, id).     */
/* The board holds (score, seq, id) sorted by (score desc, seq asc).          */
/* Returns the insertion rank, -1 if rejected, -2 if the score is non-finite. */
/* ------------------------------------------------------------------------- */

ORC_API int orc_leaderboard_update(double* scores, uint64_t* seqs, int64_t* ids, size_t* size, size_t capacity,
                                   uint64_t* seq_counter, double score, int64_t id) {
  if (!isfinite(score)) return -2;
  const uint64_t seq = (*seq_counter)++;
  size_t n = *size;
  if (n >= capacity && score <= scores[n - 1]) return -1;
  size_t pos = 0;
  while (pos < n && scores[pos] >= score) ++pos;
  size_t last = (n < capacity) ? n : capacity - 1;
  for (size_t i = last; i > pos; --i) {
    scores[i] = scores[i - 1];
    seqs[i] = seqs[i - 1];
    ids[i] = ids[i - 1];
  }
  scores[pos] = score;
  seqs[pos] = seq;
  ids[pos] = id;
  *size = (n < capacity) ? n + 1 : capacity;
  return (int)pos;
}

/* Leaderboard::refresh_stats tournament.hpp:66-87: per-coordinate mean and    */
/* population variance of the entries' flat params (entries[e] in board order).*/
ORC_API void orc_population_stats(const double* const* entries, size_t n, size_t P, double* mean, double* var) {
  if (n == 0) return; /* :69 */
  for (size_t i = 0; i < P; ++i) mean[i] = var[i] = 0.0;
  for (size_t e = 0; e < n; ++e) /* :73-76 */
    for (size_t i = 0; i < P; ++i) mean[i] += entries[e][i];
  const double inv = 1.0 / (double)n; /* :77-78 */
  for (size_t i = 0; i < P; ++i) mean[i] *= inv;
  for (size_t e = 0; e < n; ++e) /* :79-85 */
    for (size_t i = 0; i < P; ++i) {
      const double d = entries[e][i] - mean[i];
      var[i] += d * d;
    }
  for (size_t i = 0; i < P; ++i) var[i] *= inv; /* :86 */
}

/* ------------------------------------------------------------------------- */
/* Indicators: compute_indicators market.hpp:373-392 and helpers :285-366.    */
/* out[(i*K + k)*T + t] for i in macd, rsi_14, cci_30, sma_20.                */
/* ------------------------------------------------------------------------- */

static void ema(const double* x, size_t n, size_t period, double* out) { /* :289-296 */
  const double alpha = 2.0 / ((double)period + 1.0);
  if (!n) return;
  out[0] = x[0];
  for (size_t t = 1; t < n; ++t) out[t] = alpha * x[t] + (1.0 - alpha) * out[t - 1];
}

static void backfill(double* x, size_t n, size_t first) { /* :298-300 */
  for (size_t t = 0; t < first && t < n; ++t) x[t] = x[first];
}

ORC_API int orc_compute_indicators(const double* high, const double* low, const double* close, size_t T, int K,
                                   double* out) {
  if (T < 35) return 5; /* DataError, :374-378 */
  double* fast = (double*)malloc(sizeof(double) * T);
  double* slow = (double*)malloc(sizeof(double) * T);
  double* tp = (double*)malloc(sizeof(double) * T);
  for (int k = 0; k < K; ++k) {
    const double* c = close + (size_t)k * T;
    const double* h = high + (size_t)k * T;
    const double* l = low + (size_t)k * T;
    double* macd = out + ((size_t)0 * K + k) * T;
    double* rsi = out + ((size_t)1 * K + k) * T;
    double* cci = out + ((size_t)2 * K + k) * T;
    double* sma = out + ((size_t)3 * K + k) * T;
    ema(c, T, 12, fast); /* indicator_macd :302-308 */
    ema(c, T, 26, slow);
    for (size_t t = 0; t < T; ++t) macd[t] = fast[t] - slow[t];
    { /* indicator_rsi :310-333 */
      const size_t period = 14;
      for (size_t t = 0; t < T; ++t) rsi[t] = 50.0;
      double g = 0.0, ls = 0.0;
      for (size_t t = 1; t <= period; ++t) {
        const double d = c[t] - c[t - 1];
        g += maxd(d, 0.0);
        ls += maxd(-d, 0.0);
      }
      g /= (double)period;
      ls /= (double)period;
#define RSI_OF(G, L) (((G) == 0.0 && (L) == 0.0) ? 50.0 : ((L) == 0.0 ? 100.0 : 100.0 - 100.0 / (1.0 + (G) / (L))))
      rsi[period] = RSI_OF(g, ls);
      for (size_t t = period + 1; t < T; ++t) {
        const double d = c[t] - c[t - 1];
        g = (g * (double)(period - 1) + maxd(d, 0.0)) / (double)period;
        ls = (ls * (double)(period - 1) + maxd(-d, 0.0)) / (double)period;
        rsi[t] = RSI_OF(g, ls);
      }
#undef RSI_OF
      backfill(rsi, T, period);
    }
    { /* indicator_cci :335-350 */
      const size_t period = 30;
      for (size_t t = 0; t < T; ++t) tp[t] = (h[t] + l[t] + c[t]) / 3.0;
      for (size_t t = 0; t < T; ++t) cci[t] = 0.0;
      for (size_t t = period - 1; t < T; ++t) {
        double s = 0.0;
        for (size_t q = t + 1 - period; q <= t; ++q) s += tp[q];
        s /= (double)period;
        double md = 0.0;
        for (size_t q = t + 1 - period; q <= t; ++q) md += fabs(tp[q] - s);
        md /= (double)period;
        cci[t] = (md == 0.0) ? 0.0 : (tp[t] - s) / (0.015 * md);
      }
      backfill(cci, T, period - 1);
    }
    { /* indicator_sma :352-364 */
      const size_t period = 20;
      double w = 0.0;
      for (size_t t = 0; t < T; ++t) {
        sma[t] = 0.0;
        w += c[t];
        if (t >= period) w -= c[t - period];
        if (t + 1 >= period) sma[t] = w / (double)period;
      }
      backfill(sma, T, period - 1);
    }
  }
  free(fast);
  free(slow);
  free(tp);
  return 0;
}
