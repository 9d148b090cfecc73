// policy_internal.h -- launch descriptors shared by policy.cu / rollout.cu.
#pragma once
#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>

#include "mlp_simt.cuh"
#include "prb_internal.h"

enum PolicyMode : int {
  kPolicySample = 0,     // Philox noise
  kPolicyEpsIn = 1,      // injected unit normals
  kPolicyMean = 2,       // policy_mean
  kPolicyLogProb = 3,    // gaussian_log_prob of given actions
  kPolicyValueOnly = 4,  // critic only
};

struct PolicyArgs {
  const float* params;
  prb::MlpDesc actor, critic;
  int log_std_off;
  int A;
  int ldw;
  int rows_per_cta;
  int mode;
  const float* states;  // [n][S]
  size_t n;
  uint64_t seed, counter;
  const float* eps_in;
  const float* actions_in;
  float* actions;
  float* log_probs;
  float* values;
  float* eps_out;
  float* mean_out;
  float* obs_store;  // optional: first store_cols of every state row
  int store_cols;
  int32_t* status;
  // > 0: the actor MLP block (this many floats at the start of params) is bulk-copied into shared
  // memory first and the forward reads it there (a few rows per CTA: the weight walk from L2 is
  // otherwise the whole cost); 0: weights read from global memory
  int stage_actor_floats;
};

PolicyArgs prb_policy_args(prb_agent a, const float* d_states, size_t n);
size_t prb_policy_smem(const PolicyArgs& p);
void prb_policy_launch(const PolicyArgs& p, prb_ctx_s* ctx);
// P agents' policies in one launch (d_group: P PolicyArgs in device memory, rows_per_cta 32 each;
// n_max = the largest n; counter overrides every entry's Philox counter)
void prb_policy_launch_group(const PolicyArgs* d_group, int P, size_t n_max, size_t smem, uint64_t counter,
                             prb_ctx_s* ctx);
void prb_env_step_launch(prb_vecenv env, const float* d_actions, float* d_reward, uint8_t* d_done, float* d_term_obs,
                         double* d_term_ret, int32_t* d_term_len);
// One launch stepping P lock-step stock VecEnvs of one market and window (the evaluation VecEnvs of
// a GPU's pods): env p's actions at d_act + p * act_stride, its outputs at + p * n_stride.  The
// argument block (d_args, prb_env_group_args_bytes(P)) is uploaded when `upload`.  Returns false,
// doing nothing, when the envs are not such a group (the caller steps them one by one).
size_t prb_env_group_args_bytes(int P);
bool prb_env_step_group(const prb_vecenv* envs, int P, const float* d_act, size_t act_stride, float* d_rew,
                        uint8_t* d_done, double* d_tret, int32_t* d_tlen, size_t n_stride, void* d_args, bool upload);
void prb_adam_launch(prb_agent a, const float* d_grads, const int32_t* gate, cudaStream_t s);
void prb_agent_finite_gate_and_adam(prb_agent a, const float* d_grads, cudaStream_t s);
