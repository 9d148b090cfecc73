// evaluate.cu -- evaluate (pod.hpp:43-83) on device: the PodEvaluator's scoring
// of a snapshot (pod.hpp:313-316), i.e. the numbers the leaderboard ranks.
//
// The reference plays `episodes` episodes one after another on a single env,
// episode i with its own stream derive_seed(seed, kEpisode, i).  Here the
// episodes are the envs of one VecEnv, reset with exactly those streams
// (bit-exact PointMass resets) and stepped in lock-step: policy mean (or a
// Philox sample) -> clip to the spec bounds (the VecEnv step's own clamp,
// env.hpp:213-215, is the reference's std::clamp) -> env step.  An episode's
// total is the env's fp64 running return at its first done -- the same sum,
// in the same order, as the reference's `total += s.reward`.  Steps after an
// env's first done (its auto-reset continuation) are ignored.
#include <cmath>
#include <vector>

#include "policy_internal.h"
#include "prb_internal.h"

using namespace prb;

extern "C" void prb_vecenv_reset_tagged(prb_vecenv env, uint64_t seed, uint64_t tag);  // env.cu (internal)

namespace {

constexpr uint64_t kTagEpisode = 8;  // seed_tag::kEpisode common.hpp:104

__global__ void capture_first_done(size_t N, const uint8_t* __restrict__ done, const double* __restrict__ term_ret,
                                   const int32_t* __restrict__ term_len, double* __restrict__ first_ret,
                                   int32_t* __restrict__ first_len) {
  const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < N && done[i] && first_len[i] == 0) {
    first_ret[i] = term_ret[i];
    first_len[i] = term_len[i];
  }
}

// A few evaluation rows per CTA: stage the actor's weights in shared memory when they fit (the
// 64x64 stock actor: 70 KB), so the forward does not walk them from L2 (same arithmetic).
void stage_actor(PolicyArgs& p, prb_agent a) {
  if (p.actor.off[0] != 0) return;
  PolicyArgs q = p;
  q.stage_actor_floats = (int)a->Pa;
  if (prb_policy_smem(q) <= 200 * 1024) p.stage_actor_floats = (int)a->Pa;
}

}  // namespace

extern "C" {

int prb_evaluate(prb_agent a, prb_vecenv env, uint64_t seed, int sample_actions, double* episodic_rewards,
                 double* mean, double* std_dev, uint64_t* eval_steps) {
  return guard([&] {
    DeviceScope dev_(a ? a->ctx : nullptr);
    PRB_REQUIRE(a && env && episodic_rewards, PRB_ERR_USAGE, "evaluate: NULL argument");
    PRB_REQUIRE(env->N >= 1, PRB_ERR_USAGE, "evaluate: episodes must be >= 1");
    PRB_REQUIRE(a->S == env->S && a->A == env->A, PRB_ERR_DIMENSION, "evaluate: agent/env shapes disagree");
    PRB_REQUIRE(env->max_episode_steps > 0, PRB_ERR_USAGE, "evaluate: env has no episode bound");
    prb_ctx_s* ctx = env->ctx;
    cudaStream_t s = ctx->stream;
    const size_t N = env->N, A = env->A;
    // temporaries carved from the context's grow-only device scratch (no cudaMalloc / cudaFree --
    // and cudaFree's implicit device synchronisation -- per evaluation)
    auto up = [](size_t b) { return (b + 255) & ~(size_t)255; };
    const size_t o_rew = up(N * A * 4), o_lp = o_rew + up(N * 4), o_done = o_lp + up(N * 4),
                 o_tret = o_done + up(N), o_tlen = o_tret + up(N * 8), o_fret = o_tlen + up(N * 4),
                 o_flen = o_fret + up(N * 8), total = o_flen + up(N * 4);
    uint8_t* base = static_cast<uint8_t*>(ctx->device_scratch(total));
    float* act = reinterpret_cast<float*>(base);
    float* rew = reinterpret_cast<float*>(base + o_rew);
    float* lp = reinterpret_cast<float*>(base + o_lp);
    uint8_t* done = base + o_done;
    double* tret = reinterpret_cast<double*>(base + o_tret);
    int32_t* tlen = reinterpret_cast<int32_t*>(base + o_tlen);
    double* first_ret = reinterpret_cast<double*>(base + o_fret);
    int32_t* first_len = reinterpret_cast<int32_t*>(base + o_flen);
    PRB_CUDA(cudaMemsetAsync(first_len, 0, N * sizeof(int32_t), s));
    prb_vecenv_reset_tagged(env, seed, kTagEpisode);
    const uint64_t noise_seed = derive_seed(seed, {kTagEpisode});
    // every episode ends by its step limit (PointMass 200, stock: the window), so the
    // loop is bounded; the first-done capture makes later steps inert
    for (size_t step = 0; step < env->max_episode_steps; ++step) {
      PolicyArgs p = prb_policy_args(a, env->d_obs.p, N);
      stage_actor(p, a);
      if (sample_actions) {  // nn.hpp:250-265 with Philox noise (the reference draws mt19937_64 normals)
        p.mode = kPolicySample;
        p.seed = noise_seed;
        p.counter = step;
        p.actions = act;
        p.log_probs = lp;
      } else {  // policy_mean nn.hpp:268
        p.mode = kPolicyMean;
        p.mean_out = act;
      }
      p.status = nullptr;
      prb_policy_launch(p, ctx);
      prb_env_step_launch(env, act, rew, done, nullptr, tret, tlen);
      capture_first_done<<<(unsigned)((N + 255) / 256), 256, 0, s>>>(N, done, tret, tlen, first_ret,
                                                                   first_len);
      PRB_CHECK_LAUNCH();
    }
    std::vector<double> r(N);
    std::vector<int32_t> len(N);
    PRB_CUDA(cudaMemcpyAsync(r.data(), first_ret, N * sizeof(double), cudaMemcpyDeviceToHost, s));
    PRB_CUDA(cudaMemcpyAsync(len.data(), first_len, N * sizeof(int32_t), cudaMemcpyDeviceToHost, s));
    ctx->sync();
    uint64_t steps = 0;
    for (size_t i = 0; i < N; ++i) {
      PRB_REQUIRE(len[i] > 0, PRB_ERR_USAGE, "evaluate: episode " + std::to_string(i) + " did not terminate");
      steps += (uint64_t)len[i];
    }
    // EvaluationRecord: mean, population standard deviation (pod.hpp:76-81)
    const double n = (double)N;
    double m = 0.0;
    for (size_t i = 0; i < N; ++i) m += r[i];
    m /= n;
    double v = 0.0;
    for (size_t i = 0; i < N; ++i) v += (r[i] - m) * (r[i] - m);
    for (size_t i = 0; i < N; ++i) episodic_rewards[i] = r[i];
    if (mean) *mean = m;
    if (std_dev) *std_dev = std::sqrt(v / n);
    if (eval_steps) *eval_steps = steps;
  });
}

/* evaluate for the P pods of a GPU at once: every step ONE policy launch for all pods (blockIdx.y =
 * pod), then each pod's VecEnv step, then one first-done capture over all pods' episodes.  Pod p's
 * numbers equal prb_evaluate(agents[p], envs[p], seeds[p], ...) exactly (same kernels, same order
 * per episode).  episodic_rewards: [P][N]; means / std_devs / eval_steps: [P] (nullable). */
int prb_evaluate_pods(const prb_agent* agents, const prb_vecenv* envs, size_t P, const uint64_t* seeds,
                      int sample_actions, double* episodic_rewards, double* means, double* std_devs,
                      uint64_t* eval_steps) {
  return guard([&] {
    PRB_REQUIRE(agents && envs && seeds && episodic_rewards, PRB_ERR_USAGE, "evaluate_pods: NULL argument");
    if (P == 0) return;
    PRB_REQUIRE(agents[0] && envs[0], PRB_ERR_USAGE, "evaluate_pods: NULL entry");
    prb_ctx_s* ctx = envs[0]->ctx;
    DeviceScope dev_(ctx);
    const size_t N = envs[0]->N, A = envs[0]->A, T = envs[0]->max_episode_steps;
    for (size_t p = 0; p < P; ++p) {
      PRB_REQUIRE(agents[p] && envs[p], PRB_ERR_USAGE, "evaluate_pods: NULL entry");
      PRB_REQUIRE(envs[p]->N == N && envs[p]->A == A && envs[p]->max_episode_steps == T && envs[p]->ctx == ctx,
                  PRB_ERR_USAGE, "evaluate_pods: every pod's eval VecEnv needs the same shape and context");
      PRB_REQUIRE(agents[p]->S == envs[p]->S && agents[p]->A == A && agents[p]->P == agents[0]->P &&
                      agents[p]->adims == agents[0]->adims && agents[p]->cdims == agents[0]->cdims,
                  PRB_ERR_DIMENSION, "evaluate_pods: agent/env shapes disagree");
    }
    PRB_REQUIRE(N >= 1 && T > 0, PRB_ERR_USAGE, "evaluate_pods: episodes must be >= 1 and bounded");
    cudaStream_t s = ctx->stream;
    auto up = [](size_t b) { return (b + 255) & ~(size_t)255; };
    const size_t PN = P * N;
    const size_t o_rew = up(PN * A * 4), o_lp = o_rew + up(PN * 4), o_done = o_lp + up(PN * 4),
                 o_tret = o_done + up(PN), o_tlen = o_tret + up(PN * 8), o_fret = o_tlen + up(PN * 4),
                 o_flen = o_fret + up(PN * 8), o_args = o_flen + up(PN * 4), o_env = o_args + up(P * sizeof(PolicyArgs)),
                 total = o_env + up(prb_env_group_args_bytes((int)P));
    uint8_t* base = static_cast<uint8_t*>(ctx->device_scratch(total));
    float* act = reinterpret_cast<float*>(base);
    float* rew = reinterpret_cast<float*>(base + o_rew);
    float* lp = reinterpret_cast<float*>(base + o_lp);
    uint8_t* done = base + o_done;
    double* tret = reinterpret_cast<double*>(base + o_tret);
    int32_t* tlen = reinterpret_cast<int32_t*>(base + o_tlen);
    double* first_ret = reinterpret_cast<double*>(base + o_fret);
    int32_t* first_len = reinterpret_cast<int32_t*>(base + o_flen);
    PolicyArgs* d_args = reinterpret_cast<PolicyArgs*>(base + o_args);
    void* d_env_args = base + o_env;
    PRB_CUDA(cudaMemsetAsync(first_len, 0, PN * sizeof(int32_t), s));
    std::vector<PolicyArgs> args(P);
    for (size_t p = 0; p < P; ++p) {
      prb_vecenv_reset_tagged(envs[p], seeds[p], kTagEpisode);
      PolicyArgs& a = args[p];
      a = prb_policy_args(agents[p], envs[p]->d_obs.p, N);
      stage_actor(a, agents[p]);
      if (sample_actions) {
        a.mode = kPolicySample;
        a.seed = derive_seed(seeds[p], {kTagEpisode});
        a.actions = act + p * N * A;
        a.log_probs = lp + p * N;
      } else {
        a.mode = kPolicyMean;
        a.mean_out = act + p * N * A;
      }
      a.status = nullptr;
    }
    PRB_CUDA(cudaMemcpyAsync(d_args, args.data(), P * sizeof(PolicyArgs), cudaMemcpyHostToDevice, s));
    const size_t smem = prb_policy_smem(args[0]);
    bool grouped = true;  // the pods' stock eval VecEnvs step in one launch when they are lock-step
    for (size_t step = 0; step < T; ++step) {
      prb_policy_launch_group(d_args, (int)P, N, smem, step, ctx);
      if (grouped)
        grouped = prb_env_step_group(envs, (int)P, act, N * A, rew, done, tret, tlen, N, d_env_args, step == 0);
      if (!grouped)
        for (size_t p = 0; p < P; ++p)
          prb_env_step_launch(envs[p], act + p * N * A, rew + p * N, done + p * N, nullptr, tret + p * N,
                              tlen + p * N);
      capture_first_done<<<(unsigned)((PN + 255) / 256), 256, 0, s>>>(PN, done, tret, tlen, first_ret, first_len);
      PRB_CHECK_LAUNCH();
    }
    std::vector<double> r(PN);
    std::vector<int32_t> len(PN);
    PRB_CUDA(cudaMemcpyAsync(r.data(), first_ret, PN * sizeof(double), cudaMemcpyDeviceToHost, s));
    PRB_CUDA(cudaMemcpyAsync(len.data(), first_len, PN * sizeof(int32_t), cudaMemcpyDeviceToHost, s));
    ctx->sync();  // also: args (host) outlived its upload
    for (size_t p = 0; p < P; ++p) {
      uint64_t steps = 0;
      for (size_t i = 0; i < N; ++i) {
        PRB_REQUIRE(len[p * N + i] > 0, PRB_ERR_USAGE, "evaluate: episode " + std::to_string(i) + " did not terminate");
        steps += (uint64_t)len[p * N + i];
      }
      const double n = (double)N;
      double m = 0.0;
      for (size_t i = 0; i < N; ++i) m += r[p * N + i];
      m /= n;
      double v = 0.0;
      for (size_t i = 0; i < N; ++i) v += (r[p * N + i] - m) * (r[p * N + i] - m);
      for (size_t i = 0; i < N; ++i) episodic_rewards[p * N + i] = r[p * N + i];
      if (means) means[p] = m;
      if (std_devs) std_devs[p] = std::sqrt(v / n);
      if (eval_steps) eval_steps[p] = steps;
    }
  });
}

}  // extern "C"
