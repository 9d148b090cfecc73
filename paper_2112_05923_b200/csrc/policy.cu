// policy.cu -- GaussianPolicy forward + sampling + log-prob fused with the
// critic forward (nn.hpp:215-277, pod.hpp:112-113), fp32 SIMT path.
//
// One CTA owns a tile of R rows: the rows are loaded once (coalesced) into
// shared memory, pushed through the actor MLP and (optionally) the critic MLP
// with activations ping-ponging in shared memory, then each row's action
// noise is drawn from Philox4x32-10 (counter = (dim-group, row, counter)),
// a = mu + exp(log_std) * eps, and log pi(a|s) is formed exactly as
// detail::gaussian_row_log_prob (nn.hpp:215-224) but in fp32.
#include <algorithm>
#include <cmath>

#include "mlp_simt.cuh"
#include "policy_internal.h"
#include "prb_internal.h"
#include "rng.cuh"
#include "tc.cuh"

using namespace prb;

namespace {

constexpr float kLogTwoPiF = 1.8378770664093454836f;

__device__ __forceinline__ void policy_body(const PolicyArgs& p, size_t tile) {
  extern __shared__ __align__(16) float smem[];
  const int R = p.rows_per_cta;
  const int S = p.actor.dims[0];
  const int ldx = round4(S);
  float* s_x = smem;                 // [R][ldx]
  float* buf0 = s_x + R * ldx;       // [R][ldw]
  float* buf1 = buf0 + R * p.ldw;    // [R][ldw]
  float* s_mean = buf1 + R * p.ldw;  // [R][ldA]  (actor head kept for sampling)
  const int A = p.A;
  const int ldA = round4(A);
  const size_t row0 = tile * R;
  const int nrows = (p.n - row0 < (size_t)R) ? (int)(p.n - row0) : R;
  // optional staged actor weights, after the activation tiles (16-byte aligned)
  float* s_w = s_mean + ((R * ldA + 3) & ~3);
  __shared__ __align__(8) uint64_t s_wbar;
  const bool stage = p.stage_actor_floats > 0 && p.mode != kPolicyValueOnly;
  if (stage && threadIdx.x == 0) {
    tc::mbar_init(&s_wbar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    const uint32_t bytes = (uint32_t)(((size_t)p.stage_actor_floats * 4 + 15) & ~(size_t)15);
    tc::mbar_arrive_expect_tx(&s_wbar, bytes);
    tc::bulk_g2s(s_w, p.params, bytes, &s_wbar);
  }

  // ---- load the state tile (rows are contiguous in memory) ----
  {
    const float* src = p.states + row0 * S;
    const int total = nrows * S;
    int r = threadIdx.x / S, c = threadIdx.x - (threadIdx.x / S) * S;
    int bad = 0;
    for (int i = threadIdx.x; i < total; i += blockDim.x) {
      const float v = src[i];
      bad |= !isfinite(v);
      s_x[r * ldx + c] = v;
      if (p.obs_store && c < p.store_cols) p.obs_store[(row0 + r) * p.store_cols + c] = v;
      c += blockDim.x;
      while (c >= S) {
        c -= S;
        ++r;
      }
    }
    if (bad && p.status) atomicExch(p.status, PRB_ERR_NUMERIC);
  }
  __syncthreads();

  float* acts[kMaxLayers];
  int lds[kMaxLayers];
  // ---- actor ----
  if (p.mode != kPolicyValueOnly) {
    for (int l = 0; l < p.actor.nl; ++l) {
      acts[l] = (l + 1 == p.actor.nl) ? s_mean : ((l & 1) ? buf1 : buf0);
      lds[l] = (l + 1 == p.actor.nl) ? ldA : p.ldw;
    }
    if (stage) {
      __syncthreads();  // the barrier's initialisation before anyone waits on it
      tc::mbar_wait(&s_wbar, 0);
      LayerPtrs lp;
      for (int l = 0; l < p.actor.nl; ++l) {
        lp.W[l] = s_w + p.actor.off[l];
        lp.B[l] = lp.W[l] + (size_t)p.actor.dims[l] * p.actor.dims[l + 1];
        lp.ldw[l] = p.actor.dims[l + 1];
      }
      mlp_forward_tile_p(p.actor, lp, s_x, ldx, acts, lds, nrows);
    } else {
      mlp_forward_tile(p.params, p.actor, s_x, ldx, acts, lds, nrows);
    }
  }
  // ---- critic (value head) ----
  if (p.values) {
    for (int l = 0; l < p.critic.nl; ++l) {
      acts[l] = (l & 1) ? buf1 : buf0;
      lds[l] = p.ldw;
    }
    mlp_forward_tile(p.params, p.critic, s_x, ldx, acts, lds, nrows);
    const float* v = acts[p.critic.nl - 1];
    for (int r = threadIdx.x; r < nrows; r += blockDim.x) p.values[row0 + r] = v[r * p.ldw];
  }
  if (p.mode == kPolicyValueOnly) return;

  // ---- head: mean / sample / log-prob; L lanes cooperate on one row ----
  const int Q = (A + 3) / 4;  // dim groups of 4
  int L = 1;
  while (L < Q && L < 32) L <<= 1;
  const int rows_per_pass = blockDim.x / L;
  const int lane_in_row = threadIdx.x % L;
  const float* log_std = p.params + p.log_std_off;
  for (int rb = threadIdx.x / L; rb < ((nrows + rows_per_pass - 1) / rows_per_pass) * rows_per_pass;
       rb += rows_per_pass) {
    const bool active = rb < nrows;
    const size_t row = row0 + rb;
    float lp = 0.0f;
    if (active) {
      const float* mu = s_mean + rb * ldA;
      for (int q = lane_in_row; q < Q; q += L) {
        float eps4[4] = {0.f, 0.f, 0.f, 0.f};
        if (p.mode == kPolicySample) {
          const Philox4 rr = philox4x32_10((uint32_t)p.seed, (uint32_t)(p.seed >> 32), (uint32_t)q, (uint32_t)row,
                                           (uint32_t)p.counter, (uint32_t)(p.counter >> 32));
          const float2 z0 = box_muller(rr.x, rr.y), z1 = box_muller(rr.z, rr.w);
          eps4[0] = z0.x; eps4[1] = z0.y; eps4[2] = z1.x; eps4[3] = z1.y;
        }
        for (int i = 0; i < 4; ++i) {
          const int d = 4 * q + i;
          if (d >= A) break;
          const float m = mu[d];
          const float ls = log_std[d];
          float act;
          if (p.mode == kPolicyMean) {
            p.mean_out[row * A + d] = m;
            continue;
          } else if (p.mode == kPolicyLogProb) {
            act = p.actions_in[row * A + d];
          } else {
            const float e = (p.mode == kPolicyEpsIn) ? p.eps_in[row * A + d] : eps4[i];
            const float sigma = expf(ls);
            act = m + sigma * e;  // nn.hpp:260
            p.actions[row * A + d] = act;
            if (p.eps_out) p.eps_out[row * A + d] = e;
          }
          const float z = (act - m) * expf(-ls);  // (a - mu) / sigma
          lp += (-0.5f * kLogTwoPiF - ls) - 0.5f * z * z;  // nn.hpp:221-222
        }
      }
    }
    if (p.mode == kPolicyMean) continue;
    for (int o = L / 2; o > 0; o >>= 1) lp += __shfl_xor_sync(0xffffffffu, lp, o, L);
    if (active && lane_in_row == 0) p.log_probs[row] = lp;
  }
}

__global__ void __launch_bounds__(256) policy_kernel(PolicyArgs p) { policy_body(p, blockIdx.x); }

// one launch for several agents (blockIdx.y = agent): the evaluation of every pod of a GPU steps
// all pods' policies at once; counter (the Philox step) is the launch's, for every agent
__global__ void __launch_bounds__(256) policy_group_kernel(const PolicyArgs* __restrict__ group, uint64_t counter) {
  PolicyArgs p = group[blockIdx.y];
  p.counter = counter;
  if ((size_t)blockIdx.x * p.rows_per_cta < p.n) policy_body(p, blockIdx.x);
}

}  // namespace

void prb_policy_launch_group(const PolicyArgs* d_group, int P, size_t n_max, size_t smem, uint64_t counter,
                             prb_ctx_s* ctx) {
  ProfScope prof(ctx, kProfPolicy);
  if (P == 0 || n_max == 0) return;
  PRB_REQUIRE(smem <= 220 * 1024, PRB_ERR_CONFIG, "policy: tile does not fit in shared memory");
  ensure_smem(policy_group_kernel, 220 * 1024);
  const unsigned gx = (unsigned)((n_max + 31) / 32);
  policy_group_kernel<<<dim3(gx, (unsigned)P), 256, smem, ctx->stream>>>(d_group, counter);
  PRB_CHECK_LAUNCH();
}

PolicyArgs prb_policy_args(prb_agent a, const float* d_states, size_t n) {
  PolicyArgs p{};
  p.params = a->d_params.p;
  p.actor.nl = (int)a->adims.size() - 1;
  p.critic.nl = (int)a->cdims.size() - 1;
  for (size_t i = 0; i < a->adims.size(); ++i) p.actor.dims[i] = (int)a->adims[i];
  for (size_t i = 0; i < a->cdims.size(); ++i) p.critic.dims[i] = (int)a->cdims[i];
  for (size_t i = 0; i < a->aoff.size(); ++i) p.actor.off[i] = (int)a->aoff[i];
  for (size_t i = 0; i < a->coff.size(); ++i) p.critic.off[i] = (int)a->coff[i];
  p.log_std_off = (int)a->Pa;
  p.A = (int)a->A;
  int maxw = 4;
  for (size_t h : a->hidden) maxw = std::max<int>(maxw, (int)h);
  p.ldw = (maxw + 3) & ~3;
  p.states = d_states;
  p.n = n;
  p.rows_per_cta = 32;
  p.status = a->d_status.p;
  return p;
}

size_t prb_policy_smem(const PolicyArgs& p) {
  const int R = p.rows_per_cta;
  const int ldx = (p.actor.dims[0] + 3) & ~3;
  const int ldA = (p.A + 3) & ~3;
  const size_t tiles = (size_t)R * (ldx + 2 * p.ldw) + (((size_t)R * ldA + 3) & ~(size_t)3);
  return (tiles + (p.stage_actor_floats > 0 ? (((size_t)p.stage_actor_floats + 3) & ~(size_t)3) : 0)) *
         sizeof(float);
}

void prb_policy_launch(const PolicyArgs& p, prb_ctx_s* ctx) {
  cudaStream_t s = ctx->stream;
  ProfScope prof(ctx, kProfPolicy);
  if (p.n == 0) return;
  const size_t smem = prb_policy_smem(p);
  PRB_REQUIRE(smem <= 220 * 1024, PRB_ERR_CONFIG, "policy: tile does not fit in shared memory");
  ensure_smem(policy_kernel, 220 * 1024);
  const size_t grid = (p.n + p.rows_per_cta - 1) / p.rows_per_cta;
  policy_kernel<<<(unsigned)grid, 256, smem, s>>>(p);
  PRB_CHECK_LAUNCH();
}

static void finish_checked(prb_agent a, const char* what) {
  int32_t st = 0;
  PRB_CUDA(cudaMemcpyAsync(&st, a->d_status.p, sizeof(int32_t), cudaMemcpyDeviceToHost, a->ctx->stream));
  a->ctx->sync();
  if (st != 0) {
    PRB_CUDA(cudaMemsetAsync(a->d_status.p, 0, sizeof(int32_t), a->ctx->stream));
    a->ctx->sync();
    fail(PRB_ERR_NUMERIC, std::string(what) + ": non-finite entry");
  }
}

extern "C" {

int prb_policy_sample(prb_agent a, const float* d_states, size_t n, uint64_t seed, uint64_t counter, float* d_actions,
                      float* d_log_probs, float* d_values, float* d_eps) {
  return guard([&] {
    DeviceScope dev_(a ? a->ctx : nullptr);
    PRB_REQUIRE(a && d_states && d_actions && d_log_probs, PRB_ERR_USAGE, "policy_sample: NULL argument");
    PolicyArgs p = prb_policy_args(a, d_states, n);
    p.mode = kPolicySample;
    p.seed = seed;
    p.counter = counter;
    p.actions = d_actions;
    p.log_probs = d_log_probs;
    p.values = d_values;
    p.eps_out = d_eps;
    prb_policy_launch(p, a->ctx);
    finish_checked(a, "policy_sample states");  // nn.hpp:252
  });
}

int prb_policy_sample_eps(prb_agent a, const float* d_states, size_t n, const float* d_eps, float* d_actions,
                          float* d_log_probs, float* d_values) {
  return guard([&] {
    DeviceScope dev_(a ? a->ctx : nullptr);
    PRB_REQUIRE(a && d_states && d_eps && d_actions && d_log_probs, PRB_ERR_USAGE, "policy_sample: NULL argument");
    PolicyArgs p = prb_policy_args(a, d_states, n);
    p.mode = kPolicyEpsIn;
    p.eps_in = d_eps;
    p.actions = d_actions;
    p.log_probs = d_log_probs;
    p.values = d_values;
    prb_policy_launch(p, a->ctx);
    finish_checked(a, "policy_sample states");
  });
}

int prb_policy_mean(prb_agent a, const float* d_states, size_t n, float* d_mean) {
  return guard([&] {
    DeviceScope dev_(a ? a->ctx : nullptr);
    PRB_REQUIRE(a && d_states && d_mean, PRB_ERR_USAGE, "policy_mean: NULL argument");
    PolicyArgs p = prb_policy_args(a, d_states, n);
    p.mode = kPolicyMean;
    p.mean_out = d_mean;
    p.status = nullptr;
    prb_policy_launch(p, a->ctx);
    a->ctx->sync();
  });
}

int prb_policy_log_prob(prb_agent a, const float* d_states, const float* d_actions, size_t n, float* d_lp) {
  return guard([&] {
    DeviceScope dev_(a ? a->ctx : nullptr);
    PRB_REQUIRE(a && d_states && d_actions && d_lp, PRB_ERR_USAGE, "gaussian_log_prob: NULL argument");
    PolicyArgs p = prb_policy_args(a, d_states, n);
    p.mode = kPolicyLogProb;
    p.actions_in = d_actions;
    p.log_probs = d_lp;
    p.status = nullptr;
    prb_policy_launch(p, a->ctx);
    a->ctx->sync();
  });
}

int prb_critic_value(prb_agent a, const float* d_states, size_t n, float* d_values) {
  return guard([&] {
    DeviceScope dev_(a ? a->ctx : nullptr);
    PRB_REQUIRE(a && d_states && d_values, PRB_ERR_USAGE, "critic: NULL argument");
    PolicyArgs p = prb_policy_args(a, d_states, n);
    p.mode = kPolicyValueOnly;
    p.values = d_values;
    p.status = nullptr;
    prb_policy_launch(p, a->ctx);
    a->ctx->sync();
  });
}

}  // extern "C"
