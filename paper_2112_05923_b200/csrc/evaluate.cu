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
    DevBuf<float> act, rew, lp;
    DevBuf<uint8_t> done;
    DevBuf<double> tret, first_ret;
    DevBuf<int32_t> tlen, first_len;
    act.alloc(N * A);
    rew.alloc(N);
    lp.alloc(N);
    done.alloc(N);
    tret.alloc(N);
    tlen.alloc(N);
    first_ret.alloc(N);
    first_len.alloc(N);
    PRB_CUDA(cudaMemsetAsync(first_len.p, 0, first_len.bytes(), s));
    prb_vecenv_reset_tagged(env, seed, kTagEpisode);
    const uint64_t noise_seed = derive_seed(seed, {kTagEpisode});
    // every episode ends by its step limit (PointMass 200, stock: the window), so the
    // loop is bounded; the first-done capture makes later steps inert
    for (size_t step = 0; step < env->max_episode_steps; ++step) {
      PolicyArgs p = prb_policy_args(a, env->d_obs.p, N);
      if (sample_actions) {  // nn.hpp:250-265 with Philox noise (the reference draws mt19937_64 normals)
        p.mode = kPolicySample;
        p.seed = noise_seed;
        p.counter = step;
        p.actions = act.p;
        p.log_probs = lp.p;
      } else {  // policy_mean nn.hpp:268
        p.mode = kPolicyMean;
        p.mean_out = act.p;
      }
      p.status = nullptr;
      prb_policy_launch(p, ctx);
      prb_env_step_launch(env, act.p, rew.p, done.p, nullptr, tret.p, tlen.p);
      capture_first_done<<<(unsigned)((N + 255) / 256), 256, 0, s>>>(N, done.p, tret.p, tlen.p, first_ret.p,
                                                                   first_len.p);
      PRB_CHECK_LAUNCH();
    }
    std::vector<double> r(N);
    std::vector<int32_t> len(N);
    PRB_CUDA(cudaMemcpyAsync(r.data(), first_ret.p, N * sizeof(double), cudaMemcpyDeviceToHost, s));
    PRB_CUDA(cudaMemcpyAsync(len.data(), first_len.p, N * sizeof(int32_t), cudaMemcpyDeviceToHost, s));
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

}  // extern "C"
