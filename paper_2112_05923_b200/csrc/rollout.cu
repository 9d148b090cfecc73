// rollout.cu -- the device TransitionBuffer (buffer.hpp:27-135) and
// worker_collect (pod.hpp:95-132).
//
// Storage is time-major: transition (env e, step h) at h*N + e, so every step
// of the collection loop writes one contiguous slab.  For the stock env the
// 181-float observation is stored compactly: its per-env part (balance/cap,
// shares: 1+K floats) per transition, and the 5K shared features once per
// step as a time index into the env's read-only feature table (all envs of a
// VecEnv share t, stock_env.hpp:161) -- 124 B instead of 724 B per transition.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "policy_internal.h"
#include <type_traits>

#include "prb_internal.h"
#include "rollout_pm_tc.h"

using namespace prb;

namespace {

void alloc_rollout(prb_rollout_s* r) {
  const size_t cap = r->N * r->H;
  r->d_obs.alloc(cap * r->Sp + 16);  // + padding: 16-byte bulk row copies (ppo_tc.cu)
  r->d_row.alloc(r->H);
  r->d_act.alloc(cap * r->A);
  r->d_logp.alloc(cap);
  r->d_rew.alloc(cap);
  r->d_val.alloc(cap);
  r->d_adv.alloc(cap);
  r->d_ret.alloc(cap);
  r->d_done.alloc(cap);
  r->d_boot.alloc(r->N);
  r->d_advstat.alloc(2);
}

}  // namespace

bool prb_fused_rollout_supported(prb_rollout r, prb_agent a, prb_vecenv env);
void prb_tc_rollout_pods(const prb_rollout* rs, const prb_agent* as, const prb_vecenv* es, size_t P,
                         const uint64_t* seeds);
bool prb_tc_rollout_pods_supported(const prb_rollout* rs, const prb_agent* as, const prb_vecenv* es, size_t P);

// configs[2]: PointMass2D with the 3x256 actor/critic -> rollout_pm_tc.cu
static bool pm_tc_supported(prb_rollout r, prb_agent a, prb_vecenv env) {
  return r->mode == 2 && env->kind == PRB_KIND_POINTMASS && a->S == 6 && a->A == 2 && a->hidden.size() == 3 &&
         a->hidden[0] == 256 && a->hidden[1] == 256 && a->hidden[2] == 256 && r->obs_mode == 0 && r->Sp == 6;
}

static void pm_tc_collect(prb_rollout r, prb_agent a, prb_vecenv env, uint64_t seed) {
  cudaStream_t s = r->ctx->stream;
  PmPackOffsets o{};
  o.S = (int)a->S;
  o.A = (int)a->A;
  for (int i = 0; i < 4; ++i) {
    o.a_w[i] = (int)a->aoff[i];
    o.c_w[i] = (int)a->coff[i];
  }
  o.log_std = (int)a->Pa;
  if (r->d_pack.n != kPmPackBytes) r->d_pack.alloc(kPmPackBytes);
  ProfScope prof(r->ctx, kProfRollout);
  launch_pm_pack(a->d_params.p, o, r->d_pack.p, s);
  PmTcArgs t{};
  t.pack = r->d_pack.p;
  t.params = a->d_params.p;
  t.o = o;
  t.N = (int)r->N;
  t.H = (int)r->H;
  t.seed = seed;
  t.st = env->d_pm_state.p;
  t.steps = env->d_pm_steps.p;
  t.ep_return = env->d_ep_return.p;
  t.mt = env->d_mt.p;
  t.mt_idx = env->d_mt_idx.p;
  t.obs_out = env->d_obs.p;
  t.b_obs = r->d_obs.p;
  t.b_act = r->d_act.p;
  t.b_logp = r->d_logp.p;
  t.b_val = r->d_val.p;
  t.b_rew = r->d_rew.p;
  t.b_done = r->d_done.p;
  t.b_boot = r->d_boot.p;
  const char* trace_path = debug_env("PRB_PM_TRACE");  // debug: clock64 phase trace of CTA 0
  prb::DevBuf<unsigned long long> d_trace;
  if (trace_path) {
    d_trace.alloc(4 * kPmTraceLen);
    PRB_CUDA(cudaMemsetAsync(d_trace.p, 0, d_trace.bytes(), s));
    t.trace = d_trace.p;
  }
  launch_pm_rollout_tc(t, r->ctx->num_sms, s);
  if (trace_path) {
    std::vector<unsigned long long> h(4 * kPmTraceLen);
    PRB_CUDA(cudaMemcpyAsync(h.data(), d_trace.p, d_trace.bytes(), cudaMemcpyDeviceToHost, s));
    PRB_CUDA(cudaStreamSynchronize(s));
    if (FILE* f = fopen(trace_path, "wb")) {
      fwrite(h.data(), sizeof(unsigned long long), h.size(), f);
      fclose(f);
    }
  }
}
void prb_fused_rollout_launch(prb_rollout r, prb_agent a, prb_vecenv env, uint64_t seed, std::vector<int32_t>& rows);

void prb_gae_launch(prb_ctx ctx, const float* rew, const float* val, const uint8_t* done, const float* boot, size_t N,
                    size_t H, double gamma, double lambda, float* adv, float* ret, double* stat, int normalize);

extern "C" {

int prb_rollout_create(prb_vecenv env, size_t horizon, prb_rollout* out) {
  return guard([&] {
    DeviceScope dev_(env ? env->ctx : nullptr);
    PRB_REQUIRE(env && out, PRB_ERR_USAGE, "prb_rollout_create: NULL argument");
    PRB_REQUIRE(horizon > 0, PRB_ERR_CONFIG, "pod.rollout_horizon must be > 0");
    PRB_REQUIRE(env->N * horizon < ((size_t)1 << 32), PRB_ERR_CONFIG, "prb_rollout_create: N*H must be < 2^32");
    auto* r = new prb_rollout_s;
    r->ctx = env->ctx;
    r->N = env->N;
    r->H = horizon;
    r->S = env->S;
    r->A = env->A;
    if (env->kind == PRB_KIND_STOCK) {
      r->obs_mode = 1;
      r->K = env->market->K;
      r->Sp = 1 + (size_t)r->K;
      r->d_feat = env->d_feat.p;
    } else {
      r->obs_mode = 0;
      r->Sp = env->S;
    }
    alloc_rollout(r);
    *out = r;
  });
}

int prb_rollout_create_raw(prb_ctx ctx, size_t N, size_t H, size_t S, size_t A, prb_rollout* out) {
  return guard([&] {
    DeviceScope dev_(ctx);
    PRB_REQUIRE(ctx && out, PRB_ERR_USAGE, "prb_rollout_create_raw: NULL argument");
    PRB_REQUIRE(N > 0 && H > 0 && S > 0 && A > 0, PRB_ERR_CONFIG, "prb_rollout_create_raw: zero dimension");
    PRB_REQUIRE(N * H < ((size_t)1 << 32), PRB_ERR_CONFIG, "prb_rollout_create_raw: N*H must be < 2^32");
    auto* r = new prb_rollout_s;
    r->ctx = ctx;
    r->N = N;
    r->H = H;
    r->S = S;
    r->A = A;
    r->obs_mode = 0;
    r->Sp = S;
    alloc_rollout(r);
    *out = r;
  });
}

int prb_rollout_destroy(prb_rollout r) {
  return guard([&] {
    DeviceScope dev_(r ? r->ctx : nullptr);
    if (r) cudaStreamSynchronize(r->ctx->stream);
    delete r;
  });
}

int prb_rollout_collect(prb_rollout r, prb_agent a, prb_vecenv env, uint64_t seed) {
  return guard([&] {
    DeviceScope dev_(a ? a->ctx : nullptr);
    PRB_REQUIRE(r && a && env, PRB_ERR_USAGE, "worker_collect: NULL argument");
    PRB_REQUIRE(env->N == r->N && env->S == r->S && env->A == r->A && a->S == env->S && a->A == env->A,
                PRB_ERR_USAGE, "worker_collect: rollout/agent/env shapes disagree");
    PRB_REQUIRE(env->was_reset, PRB_ERR_DIMENSION, "vec_step: sub-environments have no state (call reset first)");
    const bool compact = env->kind == PRB_KIND_STOCK;
    if (compact) {
      if (r->obs_mode != 1) {  // an upload switched the buffer to full rows; switch back
        r->obs_mode = 1;
        r->K = env->market->K;
        r->Sp = 1 + (size_t)r->K;
        r->d_obs.alloc(r->N * r->H * r->Sp + 16);
      }
      r->d_feat = env->d_feat.p;
    }
    cudaStream_t s = r->ctx->stream;
    const size_t N = r->N, H = r->H, A = r->A;
    std::vector<int32_t> rows(H);
    if (pm_tc_supported(r, a, env)) {
      pm_tc_collect(r, a, env, seed);
      r->ctx->sync();
      r->full = true;
      r->gae_valid = false;
      return;
    }
    if (r->mode != 0 && prb_fused_rollout_supported(r, a, env)) {
      prb_fused_rollout_launch(r, a, env, seed, rows);
      PRB_CUDA(cudaMemcpyAsync(r->d_row.p, rows.data(), H * sizeof(int32_t), cudaMemcpyHostToDevice, s));
      r->ctx->sync();
      r->full = true;
      r->gae_valid = false;
      return;
    }
    for (size_t h = 0; h < H; ++h) {
      if (compact) rows[h] = (int32_t)env->t;
      PolicyArgs p = prb_policy_args(a, env->d_obs.p, N);
      p.mode = kPolicySample;
      p.seed = seed;
      p.counter = h;
      p.actions = r->d_act.p + h * N * A;
      p.log_probs = r->d_logp.p + h * N;
      p.values = r->d_val.p + h * N;
      p.obs_store = r->d_obs.p + h * N * r->Sp;
      p.store_cols = (int)r->Sp;
      p.status = nullptr;
      prb_policy_launch(p, r->ctx);
      prb_env_step_launch(env, p.actions, r->d_rew.p + h * N, r->d_done.p + h * N, nullptr, nullptr, nullptr);
    }
    // bootstrap V(s_H) (pod.hpp:127-131)
    PolicyArgs p = prb_policy_args(a, env->d_obs.p, N);
    p.mode = kPolicyValueOnly;
    p.values = r->d_boot.p;
    p.status = nullptr;
    prb_policy_launch(p, r->ctx);
    if (compact) PRB_CUDA(cudaMemcpyAsync(r->d_row.p, rows.data(), H * sizeof(int32_t), cudaMemcpyHostToDevice, s));
    r->ctx->sync();  // rows[] lives on this stack frame
    r->full = true;
    r->gae_valid = false;
  });
}

int prb_rollout_collect_pods(const prb_rollout* rs, const prb_agent* as, const prb_vecenv* es, size_t P,
                             const uint64_t* seeds) {
  return guard([&] {
    PRB_REQUIRE(rs && as && es && seeds && P > 0, PRB_ERR_USAGE, "worker_collect (pods): NULL argument");
    for (size_t p = 0; p < P; ++p) {
      PRB_REQUIRE(rs[p] && as[p] && es[p], PRB_ERR_USAGE, "worker_collect (pods): NULL argument");
      PRB_REQUIRE(rs[p]->ctx->device == rs[0]->ctx->device && as[p]->ctx->device == rs[0]->ctx->device,
                  PRB_ERR_USAGE, "worker_collect (pods): pods on different devices");
      PRB_REQUIRE(es[p]->N == rs[p]->N && es[p]->S == rs[p]->S && es[p]->A == rs[p]->A && as[p]->S == es[p]->S &&
                      as[p]->A == es[p]->A,
                  PRB_ERR_USAGE, "worker_collect: rollout/agent/env shapes disagree");
      for (size_t q = 0; q < p; ++q)
        PRB_REQUIRE(rs[q] != rs[p] && es[q] != es[p], PRB_ERR_USAGE,
                    "worker_collect (pods): a rollout or VecEnv appears twice");
      if (es[p]->kind == PRB_KIND_STOCK && rs[p]->obs_mode != 1) {  // back to compact rows after an upload
        rs[p]->obs_mode = 1;
        rs[p]->K = es[p]->market->K;
        rs[p]->Sp = 1 + (size_t)rs[p]->K;
        rs[p]->d_obs.alloc(rs[p]->N * rs[p]->H * rs[p]->Sp + 16);
      }
    }
    DeviceScope dev_(rs[0]->ctx);
    if (!prb_tc_rollout_pods_supported(rs, as, es, P)) {  // other envs / nets: one collect per pod
      for (size_t p = 0; p < P; ++p) {
        const int rc = prb_rollout_collect(rs[p], as[p], es[p], seeds[p]);
        if (rc) fail(rc, prb_last_error());
      }
      return;
    }
    prb_tc_rollout_pods(rs, as, es, P, seeds);
    for (size_t p = 0; p < P; ++p) {
      rs[p]->full = true;
      rs[p]->gae_valid = false;
    }
  });
}

int prb_rollout_set_mode(prb_rollout r, int mode) {
  return guard([&] {
    DeviceScope dev_(r ? r->ctx : nullptr);
    PRB_REQUIRE(r, PRB_ERR_USAGE, "prb_rollout_set_mode: NULL rollout");
    PRB_REQUIRE(mode >= 0 && mode <= 2, PRB_ERR_CONFIG, "prb_rollout_set_mode: mode must be 0, 1 or 2");
    r->mode = mode;
  });
}

int prb_rollout_device_fields(prb_rollout r, float** d_obs, float** d_actions, float** d_log_probs, float** d_rewards,
                              float** d_values, uint8_t** d_dones, float** d_bootstrap) {
  return guard([&] {
    DeviceScope dev_(r ? r->ctx : nullptr);
    PRB_REQUIRE(r, PRB_ERR_USAGE, "prb_rollout_device_fields: NULL rollout");
    if (d_obs) *d_obs = r->d_obs.p;
    if (d_actions) *d_actions = r->d_act.p;
    if (d_log_probs) *d_log_probs = r->d_logp.p;
    if (d_rewards) *d_rewards = r->d_rew.p;
    if (d_values) *d_values = r->d_val.p;
    if (d_dones) *d_dones = r->d_done.p;
    if (d_bootstrap) *d_bootstrap = r->d_boot.p;
  });
}

int prb_rollout_download(prb_rollout r, double* states, double* actions, double* log_probs, double* rewards,
                         uint8_t* dones, double* values, double* bootstrap) {
  return guard([&] {
    DeviceScope dev_(r ? r->ctx : nullptr);
    PRB_REQUIRE(r, PRB_ERR_USAGE, "prb_rollout_download: NULL rollout");
    const size_t N = r->N, H = r->H, n = N * H, S = r->S, A = r->A, Sp = r->Sp;
    cudaStream_t s = r->ctx->stream;
    auto pull = [&](const auto* d, size_t count, auto& h) {
      h.resize(count);
      PRB_CUDA(cudaMemcpyAsync(h.data(), d, count * sizeof(*d), cudaMemcpyDeviceToHost, s));
    };
    std::vector<float> obs, act, lp, rw, vl, bt, feat;
    std::vector<uint8_t> dn;
    std::vector<int32_t> rows;
    if (states) pull(r->d_obs.p, n * Sp, obs);
    if (states && r->obs_mode == 1) {
      pull(r->d_row.p, H, rows);
      r->ctx->sync();
      int32_t tmax = 0;
      for (int32_t t : rows) tmax = std::max(tmax, t);
      pull(r->d_feat, (size_t)(tmax + 1) * 5 * r->K, feat);
    }
    if (actions) pull(r->d_act.p, n * A, act);
    if (log_probs) pull(r->d_logp.p, n, lp);
    if (rewards) pull(r->d_rew.p, n, rw);
    if (values) pull(r->d_val.p, n, vl);
    if (dones) pull(r->d_done.p, n, dn);
    if (bootstrap) pull(r->d_boot.p, N, bt);
    r->ctx->sync();
    const size_t F = 5 * (size_t)r->K;
    for (size_t e = 0; e < N; ++e)
      for (size_t h = 0; h < H; ++h) {
        const size_t j = h * N + e, i = e * H + h;  // device time-major -> reference env-major
        if (states) {
          for (size_t c = 0; c < Sp; ++c) states[i * S + c] = obs[j * Sp + c];
          if (r->obs_mode == 1)
            for (size_t c = 0; c < F; ++c) states[i * S + Sp + c] = feat[(size_t)rows[h] * F + c];
        }
        if (actions)
          for (size_t c = 0; c < A; ++c) actions[i * A + c] = act[j * A + c];
        if (log_probs) log_probs[i] = lp[j];
        if (rewards) rewards[i] = rw[j];
        if (values) values[i] = vl[j];
        if (dones) dones[i] = dn[j];
      }
    if (bootstrap)
      for (size_t e = 0; e < N; ++e) bootstrap[e] = bt[e];
  });
}

int prb_rollout_download_chunks(prb_rollout r, const uint64_t* envs, size_t n_envs, double* states, double* actions,
                                double* log_probs, double* rewards, uint8_t* dones, double* values, double* bootstrap,
                                double* raw_advantages, double* returns) {
  return guard([&] {
    DeviceScope dev_(r ? r->ctx : nullptr);
    PRB_REQUIRE(r && (envs || n_envs == 0), PRB_ERR_USAGE, "prb_rollout_download_chunks: NULL argument");
    PRB_REQUIRE(!(raw_advantages || returns) || r->gae_valid, PRB_ERR_USAGE,
                "prb_rollout_download_chunks: advantages requested before prb_gae");
    const size_t N = r->N, H = r->H, S = r->S, A = r->A, Sp = r->Sp;
    for (size_t i = 0; i < n_envs; ++i)
      PRB_REQUIRE(envs[i] < N, PRB_ERR_USAGE, "prb_rollout_download_chunks: env index out of range");
    cudaStream_t s = r->ctx->stream;
    // one strided copy per (env, field): H rows of w elements at pitch N * w (time-major buffer)
    auto column = [&](const auto* d, size_t w, size_t e, auto* h) {
      using T = std::remove_const_t<std::remove_pointer_t<decltype(d)>>;
      PRB_CUDA(cudaMemcpy2DAsync(h, w * sizeof(T), d + e * w, N * w * sizeof(T), w * sizeof(T), H,
                                 cudaMemcpyDeviceToHost, s));
    };
    std::vector<float> obs(states ? n_envs * H * Sp : 0), act(actions ? n_envs * H * A : 0);
    std::vector<float> lp(log_probs ? n_envs * H : 0), rw(rewards ? n_envs * H : 0), vl(values ? n_envs * H : 0);
    std::vector<float> ad(raw_advantages ? n_envs * H : 0), rt(returns ? n_envs * H : 0), bt(bootstrap ? n_envs : 0);
    std::vector<uint8_t> dn(dones ? n_envs * H : 0);
    for (size_t i = 0; i < n_envs; ++i) {
      const size_t e = envs[i];
      if (states) column(r->d_obs.p, Sp, e, obs.data() + i * H * Sp);
      if (actions) column(r->d_act.p, A, e, act.data() + i * H * A);
      if (log_probs) column(r->d_logp.p, 1, e, lp.data() + i * H);
      if (rewards) column(r->d_rew.p, 1, e, rw.data() + i * H);
      if (values) column(r->d_val.p, 1, e, vl.data() + i * H);
      if (dones) column(r->d_done.p, 1, e, dn.data() + i * H);
      if (raw_advantages) column(r->d_adv.p, 1, e, ad.data() + i * H);
      if (returns) column(r->d_ret.p, 1, e, rt.data() + i * H);
      if (bootstrap) PRB_CUDA(cudaMemcpyAsync(bt.data() + i, r->d_boot.p + e, sizeof(float), cudaMemcpyDeviceToHost, s));
    }
    std::vector<int32_t> rows;
    std::vector<float> feat;
    const size_t F = 5 * (size_t)r->K;
    if (states && r->obs_mode == 1) {
      rows.resize(H);
      PRB_CUDA(cudaMemcpyAsync(rows.data(), r->d_row.p, H * sizeof(int32_t), cudaMemcpyDeviceToHost, s));
      r->ctx->sync();
      int32_t tmax = 0;
      for (int32_t t : rows) tmax = std::max(tmax, t);
      feat.resize((size_t)(tmax + 1) * F);
      PRB_CUDA(cudaMemcpyAsync(feat.data(), r->d_feat, feat.size() * sizeof(float), cudaMemcpyDeviceToHost, s));
    }
    r->ctx->sync();
    for (size_t i = 0; i < n_envs; ++i)
      for (size_t h = 0; h < H; ++h) {
        const size_t j = i * H + h;  // output row: chunk i, step h (the reference's e*H + h order)
        if (states) {
          for (size_t c = 0; c < Sp; ++c) states[j * S + c] = obs[j * Sp + c];
          if (r->obs_mode == 1)
            for (size_t c = 0; c < F; ++c) states[j * S + Sp + c] = feat[(size_t)rows[h] * F + c];
        }
        if (actions)
          for (size_t c = 0; c < A; ++c) actions[j * A + c] = act[j * A + c];
        if (log_probs) log_probs[j] = lp[j];
        if (rewards) rewards[j] = rw[j];
        if (values) values[j] = vl[j];
        if (dones) dones[j] = dn[j];
        if (raw_advantages) raw_advantages[j] = ad[j];
        if (returns) returns[j] = rt[j];
      }
    for (size_t i = 0; i < n_envs && bootstrap; ++i) bootstrap[i] = bt[i];
  });
}

int prb_rollout_upload(prb_rollout r, const double* states, const double* actions, const double* log_probs,
                       const double* rewards, const uint8_t* dones, const double* values, const double* bootstrap) {
  return guard([&] {
    DeviceScope dev_(r ? r->ctx : nullptr);
    PRB_REQUIRE(r && states && actions && log_probs && rewards && dones && values && bootstrap, PRB_ERR_USAGE,
                "prb_rollout_upload: NULL argument");
    const size_t N = r->N, H = r->H, n = N * H, S = r->S, A = r->A;
    if (r->obs_mode != 0) {
      r->obs_mode = 0;
      r->Sp = S;
      r->d_obs.alloc(n * S + 16);
    }
    std::vector<float> obs(n * S), act(n * A), lp(n), rw(n), vl(n), bt(N);
    std::vector<uint8_t> dn(n);
    for (size_t e = 0; e < N; ++e)
      for (size_t h = 0; h < H; ++h) {
        const size_t j = h * N + e, i = e * H + h;
        for (size_t c = 0; c < S; ++c) obs[j * S + c] = (float)states[i * S + c];
        for (size_t c = 0; c < A; ++c) act[j * A + c] = (float)actions[i * A + c];
        lp[j] = (float)log_probs[i];
        rw[j] = (float)rewards[i];
        vl[j] = (float)values[i];
        dn[j] = dones[i] ? 1 : 0;
      }
    for (size_t e = 0; e < N; ++e) bt[e] = (float)bootstrap[e];
    cudaStream_t s = r->ctx->stream;
    PRB_CUDA(cudaMemcpyAsync(r->d_obs.p, obs.data(), obs.size() * sizeof(float), cudaMemcpyHostToDevice, s));
    PRB_CUDA(cudaMemcpyAsync(r->d_act.p, act.data(), act.size() * sizeof(float), cudaMemcpyHostToDevice, s));
    PRB_CUDA(cudaMemcpyAsync(r->d_logp.p, lp.data(), n * sizeof(float), cudaMemcpyHostToDevice, s));
    PRB_CUDA(cudaMemcpyAsync(r->d_rew.p, rw.data(), n * sizeof(float), cudaMemcpyHostToDevice, s));
    PRB_CUDA(cudaMemcpyAsync(r->d_val.p, vl.data(), n * sizeof(float), cudaMemcpyHostToDevice, s));
    PRB_CUDA(cudaMemcpyAsync(r->d_done.p, dn.data(), n, cudaMemcpyHostToDevice, s));
    PRB_CUDA(cudaMemcpyAsync(r->d_boot.p, bt.data(), N * sizeof(float), cudaMemcpyHostToDevice, s));
    r->ctx->sync();
    r->full = true;
    r->gae_valid = false;
  });
}

}  // extern "C"
