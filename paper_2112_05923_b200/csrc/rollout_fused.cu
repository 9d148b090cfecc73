// rollout_fused.cu -- worker_collect (pod.hpp:95-132) for the stock-trading
// VecEnv as ONE persistent kernel per rollout: each CTA owns a tile of
// kRows envs for all H steps, keeps their portfolio state (fp64 balance,
// int32 shares, fp64 episode return) and all actor/critic weights on chip, and
// per step runs
//   obs -> actor/critic MLP (fp32 SIMT, register-tiled, weights in smem)
//       -> Philox Gaussian sample + log-prob -> stock_env_step (fp64)
//       -> coalesced writes of the compact rollout rows.
// HBM traffic per transition is only the rollout buffer (257 B): the obs is
// never materialised (its 150 shared features are a per-step constant).
//
// Lock-step algebra: every env of a VecEnv sits at the same
// t, so the first layer's contribution of the 150 shared features,
// feat[t] . W1[31:181], is the same for all envs; it is computed once per step
// (shared_layer1_kernel) and the per-env first layer is a 31-wide product.
// The result is the same function; only fp32 summation order differs.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cmath>

#include "policy_internal.h"
#include "prb_internal.h"
#include "rng.cuh"
#include "stock_env.cuh"
#include "rollout_tc.h"

using namespace prb;

namespace {

constexpr int kRows = 32;      // envs per CTA
constexpr int kThreads = 256;
constexpr int kH1 = 64, kH2 = 64;
constexpr int kXW = 32;        // private obs width padded (1 + K <= 32)
constexpr float kLogTwoPiF = 1.8378770664093454836f;

struct FusedArgs {
  const float* __restrict__ params;
  int a_w1, a_w2, a_w3, c_w1, c_w2, c_w3, log_std;  // flat offsets (W; b follows)
  int S, K;
  const float* __restrict__ shared_l1;  // [H+1][128] feat[t_h] . W1[31:] (actor 0-63, critic 64-127)
  const int32_t* __restrict__ t_seq;    // [H+1] portfolio t before step h
  const uint8_t* __restrict__ done_seq; // [H]
  const double* __restrict__ close_tk;  // [T][K]
  const float* __restrict__ feat;       // [T][5K]
  double cap, max_trade, cost;
  int N, H, start, ep_len0;             // ep_len0 = step_count before step 0
  uint64_t seed;
  double* __restrict__ balance;
  int32_t* __restrict__ shares;  // [K][N]
  double* __restrict__ ep_return;
  float* __restrict__ obs_out;   // [N][S] final states
  float* __restrict__ b_obs;     // [H][N][1+K]
  float* __restrict__ b_act;     // [H][N][K]
  float* __restrict__ b_logp;    // [H][N]
  float* __restrict__ b_val;
  float* __restrict__ b_rew;
  uint8_t* __restrict__ b_done;
  float* __restrict__ b_boot;    // [N]
};

__device__ __forceinline__ double clamp_ref(double v, double lo, double hi) { return (v < lo) ? lo : ((hi < v) ? hi : v); }
__device__ __forceinline__ double min_ref(double a, double b) { return (b < a) ? b : a; }
__device__ __forceinline__ double max_ref(double a, double b) { return (a < b) ? b : a; }

struct Smem {
  float W1p[kXW][128];      // private rows of layer 1, actor | critic
  float W2[2][kH1][kH2];    // actor, critic
  float W3[kH2][32];        // actor head cols 0..A-1 (others 0)
  float W3c[kH2];           // critic head
  float b1[128], b2[128], b3[32], ls[32], sig[32];
  float b3c;
  alignas(16) float x[kRows][kXW];  // float4-read operands must stay 16-byte aligned
  alignas(16) float h1[kRows][128];
  alignas(16) float h2[kRows][128];
  alignas(16) float head[kRows][32];    // mean 0..A-1, value at 31
  alignas(16) float act[kRows][32];
  double bal[kRows], ret[kRows];
  double p0[kXW], p1[kXW];
  int32_t sh[kXW][kRows];
  float lp[kRows];
  float rew[kRows];
};

// s_out[r][c] = act(bias[c] + pre[c] + sum_k s_in[r][k] W[k][c]) ; 128 output columns,
// actor (c < 64) / critic (c >= 64) each with its own weights & input half when SPLIT.
template <int KIN, bool SPLIT>
__device__ __forceinline__ void layer128(const float (*in)[128], const float* in_flat, int ldi, const float* W0,
                                         const float* W1, int ldw, const float* bias, const float* pre,
                                         float (*out)[128]) {
  const int t = threadIdx.x;
  const int cg = t & 31;  // 4 columns
  const int rg = t >> 5;  // 4 rows: rg*4 .. rg*4+3
  const int c0 = cg * 4;
  const bool critic = SPLIT && c0 >= 64;
  const float* W = critic ? W1 : W0;
  const int wc = critic ? c0 - 64 : c0;
  const int ioff = critic ? 64 : 0;
  float acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0.f;
  const float* xin = in_flat + (rg * 4) * ldi + ioff;
#pragma unroll 4
  for (int k = 0; k < KIN; k += 4) {
    float4 w[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) w[q] = *reinterpret_cast<const float4*>(W + (k + q) * ldw + wc);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const float4 xv = *reinterpret_cast<const float4*>(xin + i * ldi + k);
      const float xs[4] = {xv.x, xv.y, xv.z, xv.w};
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        acc[i][0] = fmaf(xs[q], w[q].x, acc[i][0]);
        acc[i][1] = fmaf(xs[q], w[q].y, acc[i][1]);
        acc[i][2] = fmaf(xs[q], w[q].z, acc[i][2]);
        acc[i][3] = fmaf(xs[q], w[q].w, acc[i][3]);
      }
    }
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    float4 o;
    float* op = &o.x;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      float z = acc[i][j];
      if (pre) z += pre[c0 + j];
      z += bias[c0 + j];
      op[j] = tanhf(z);
    }
    *reinterpret_cast<float4*>(&out[rg * 4 + i][c0]) = o;
  }
}

__global__ void __launch_bounds__(kThreads, 2) stock_rollout_fused_kernel(FusedArgs a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  Smem& s = *reinterpret_cast<Smem*>(smem_raw);
  const int tid = threadIdx.x;
  const int K = a.K, A = a.K, P1 = 1 + a.K, F = 5 * a.K;
  const size_t e0 = (size_t)blockIdx.x * kRows;
  const int nloc = min(kRows, a.N - (int)e0);

  // ---- weights -> smem (once per rollout) ----
  const float* P = a.params;
  for (int i = tid; i < kXW * 128; i += kThreads) {
    const int k = i / 128, c = i % 128;
    float v = 0.f;
    if (k < P1) v = (c < 64) ? P[a.a_w1 + k * kH1 + c] : P[a.c_w1 + k * kH1 + (c - 64)];
    s.W1p[k][c] = v;
  }
  for (int i = tid; i < 2 * kH1 * kH2; i += kThreads) {
    const int n = i / (kH1 * kH2), r = i % (kH1 * kH2);
    s.W2[n][r / kH2][r % kH2] = P[(n ? a.c_w2 : a.a_w2) + r];
  }
  for (int i = tid; i < kH2 * 32; i += kThreads) {
    const int k = i / 32, c = i % 32;
    s.W3[k][c] = (c < A) ? P[a.a_w3 + k * A + c] : 0.f;
  }
  for (int i = tid; i < kH2; i += kThreads) s.W3c[i] = P[a.c_w3 + i];
  for (int i = tid; i < 128; i += kThreads) {
    s.b1[i] = (i < 64) ? P[a.a_w1 + a.S * kH1 + i] : P[a.c_w1 + a.S * kH1 + i - 64];
    s.b2[i] = (i < 64) ? P[a.a_w2 + kH1 * kH2 + i] : P[a.c_w2 + kH1 * kH2 + i - 64];
  }
  for (int i = tid; i < 32; i += kThreads) {
    s.b3[i] = (i < A) ? P[a.a_w3 + kH2 * A + i] : 0.f;
    const float l = (i < A) ? P[a.log_std + i] : 0.f;
    s.ls[i] = l;
    s.sig[i] = expf(l);
  }
  if (tid == 0) s.b3c = P[a.c_w3 + kH2];
  // ---- env state -> smem ----
  if (tid < kRows) {
    const bool on = tid < nloc;
    s.bal[tid] = on ? a.balance[e0 + tid] : a.cap;
    s.ret[tid] = on ? a.ep_return[e0 + tid] : 0.0;
  }
  for (int i = tid; i < K * kRows; i += kThreads) {
    const int k = i / kRows, r = i % kRows;
    s.sh[k][r] = (r < nloc) ? a.shares[(size_t)k * a.N + e0 + r] : 0;
  }
  __syncthreads();

  for (int h = 0; h <= a.H; ++h) {
    const int t = a.t_seq[h];
    // ---- private obs row x = [balance/cap, shares] (stock_observation stock_env.hpp:115-121) ----
    for (int i = tid; i < kRows * kXW; i += kThreads) {
      const int r = i / kXW, c = i % kXW;
      float v = 0.f;
      if (c == 0) v = (float)__ddiv_rn(s.bal[r], a.cap);
      else if (c < P1) v = (float)s.sh[c - 1][r];
      s.x[r][c] = v;
    }
    if (tid < K) {
      s.p0[tid] = a.close_tk[(size_t)t * K + tid];
      if (h < a.H) s.p1[tid] = a.close_tk[(size_t)(t + 1) * K + tid];
    }
    __syncthreads();
    if (h < a.H) {  // compact obs rows of step h (contiguous span for this CTA)
      float* dst = a.b_obs + ((size_t)h * a.N + e0) * P1;
      for (int i = tid; i < nloc * P1; i += kThreads) dst[i] = s.x[i / P1][i % P1];
    }
    // ---- layer 1: 31-wide private product + per-step shared-feature term ----
    layer128<kXW, false>(nullptr, &s.x[0][0], kXW, &s.W1p[0][0], nullptr, 128, s.b1, a.shared_l1 + (size_t)h * 128,
                         s.h1);
    __syncthreads();
    // ---- layer 2: actor | critic ----
    layer128<kH1, true>(s.h1, &s.h1[0][0], 128, &s.W2[0][0][0], &s.W2[1][0][0], kH2, s.b2, nullptr, s.h2);
    __syncthreads();
    // ---- layer 3: actor mean (cols < A) and critic value (col 31) ----
    {
      const int c = tid & 31;
      const int rb = tid >> 5;  // rows rb, rb+8, rb+16, rb+24
      const bool val = (c == 31);
      float acc[4] = {0.f, 0.f, 0.f, 0.f};
      const int ioff = val ? 64 : 0;
#pragma unroll 8
      for (int k = 0; k < kH2; ++k) {
        const float w = val ? s.W3c[k] : s.W3[k][c];
#pragma unroll
        for (int i = 0; i < 4; ++i) acc[i] = fmaf(s.h2[rb + 8 * i][ioff + k], w, acc[i]);
      }
#pragma unroll
      for (int i = 0; i < 4; ++i) s.head[rb + 8 * i][c] = acc[i] + (val ? s.b3c : s.b3[c]);
    }
    __syncthreads();
    if (h == a.H) {  // bootstrap V(s_H) (pod.hpp:127-131) and the VecEnv's final states
      if (tid < nloc) a.b_boot[e0 + tid] = s.head[tid][31];
      const float* fr = a.feat + (size_t)t * F;
      float* dst = a.obs_out + e0 * a.S;
      for (int i = tid; i < nloc * a.S; i += kThreads) {
        const int r = i / a.S, c = i % a.S;
        dst[i] = (c < P1) ? s.x[r][c] : fr[c - P1];
      }
      break;
    }
    // ---- sample a = mu + sigma*eps (Philox, same stream as policy_kernel), log-prob ----
    {
      const int r = tid >> 3;       // 32 rows x 8 lanes
      const int lane8 = tid & 7;    // dim group q = lane8 (4 dims each)
      float lp = 0.f;
      const int q = lane8;
      if (4 * q < A && r < nloc) {
        const uint32_t row = (uint32_t)(e0 + r);
        const Philox4 rr = philox4x32_10((uint32_t)a.seed, (uint32_t)(a.seed >> 32), (uint32_t)q, row,
                                         (uint32_t)h, 0u);
        const float2 z0 = box_muller(rr.x, rr.y), z1 = box_muller(rr.z, rr.w);
        const float e4[4] = {z0.x, z0.y, z1.x, z1.y};
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int d = 4 * q + i;
          if (d < A) {
            const float m = s.head[r][d];
            const float act = m + s.sig[d] * e4[i];
            s.act[r][d] = act;
            const float z = (act - m) / s.sig[d];
            lp += (-0.5f * kLogTwoPiF - s.ls[d]) - 0.5f * z * z;
          }
        }
      }
      lp += __shfl_xor_sync(0xffffffffu, lp, 4, 8);
      lp += __shfl_xor_sync(0xffffffffu, lp, 2, 8);
      lp += __shfl_xor_sync(0xffffffffu, lp, 1, 8);
      if (lane8 == 0) s.lp[r] = lp;
    }
    __syncthreads();
    // ---- env step (stock_env_step stock_env.hpp:55-103), one thread per env, fp64 ----
    const int done = a.done_seq[h];
    if (tid < kRows) {
      const int r = tid;
      double bal = s.bal[r];
      double vb = bal;
      for (int k = 0; k < K; ++k) vb = __dadd_rn(vb, __dmul_rn((double)s.sh[k][r], s.p0[k]));
      for (int k = 0; k < K; ++k) {
        const double d = trunc(__dmul_rn(clamp_ref((double)s.act[r][k], -1.0, 1.0), a.max_trade));
        if (d < 0.0) {
          const int32_t held = s.sh[k][r];
          const double qv = -min_ref(-d, (double)held);
          const double price = s.p0[k];
          const double cost = __dmul_rn(__dmul_rn(a.cost, fabs(qv)), price);
          bal = __dsub_rn(bal, __dadd_rn(__dmul_rn(qv, price), cost));
          s.sh[k][r] = held + (int32_t)qv;
        }
      }
      const double cf = __dadd_rn(1.0, a.cost);
      for (int k = 0; k < K; ++k) {
        const double d = trunc(__dmul_rn(clamp_ref((double)s.act[r][k], -1.0, 1.0), a.max_trade));
        if (d > 0.0) {
          const double price = s.p0[k];
          const double qv = stock::buy_qty(d, bal, __dmul_rn(price, cf));
          const double cost = __dmul_rn(__dmul_rn(a.cost, fabs(qv)), price);
          bal = __dsub_rn(bal, __dadd_rn(__dmul_rn(qv, price), cost));
          s.sh[k][r] += (int32_t)qv;
        }
      }
      double va = bal;
      for (int k = 0; k < K; ++k) va = __dadd_rn(va, __dmul_rn((double)s.sh[k][r], s.p1[k]));
      const double rw = __dsub_rn(va, vb);
      s.rew[r] = (float)rw;
      const double ret = __dadd_rn(s.ret[r], rw);
      if (done) {  // auto-reset (env.hpp:221-229, stock_env.hpp:158-163)
        s.bal[r] = a.cap;
        s.ret[r] = 0.0;
        for (int k = 0; k < K; ++k) s.sh[k][r] = 0;
      } else {
        s.bal[r] = bal;
        s.ret[r] = ret;
      }
    }
    __syncthreads();
    // ---- coalesced rollout writes of step h ----
    {
      const size_t slab = (size_t)h * a.N + e0;
      float* da = a.b_act + slab * A;
      for (int i = tid; i < nloc * A; i += kThreads) da[i] = s.act[i / A][i % A];
      if (tid < nloc) {
        a.b_logp[slab + tid] = s.lp[tid];
        a.b_val[slab + tid] = s.head[tid][31];
        a.b_rew[slab + tid] = s.rew[tid];
        a.b_done[slab + tid] = (uint8_t)done;
      }
    }
    // (the next iteration's first __syncthreads orders these smem reads before reuse)
  }
  // ---- portfolio state back to HBM ----
  __syncthreads();
  if (tid < nloc) {
    a.balance[e0 + tid] = s.bal[tid];
    a.ep_return[e0 + tid] = s.ret[tid];
  }
  for (int i = tid; i < K * kRows; i += kThreads) {
    const int k = i / kRows, r = i % kRows;
    if (r < nloc) a.shares[(size_t)k * a.N + e0 + r] = s.sh[k][r];
  }
}

// shared_l1[h][c] = sum_{i<5K} feat[t_h][i] * W1[1+K+i][c]  (actor c<64, critic c>=64)
__global__ void shared_layer1_kernel(const float* __restrict__ params, int a_w1, int c_w1, int P1, int F,
                                     const float* __restrict__ feat, const int32_t* __restrict__ t_seq,
                                     float* __restrict__ out) {
  const int h = blockIdx.x, c = threadIdx.x;  // 128 threads
  const float* fr = feat + (size_t)t_seq[h] * F;
  const float* W = params + ((c < 64) ? a_w1 : c_w1);
  const int cc = c & 63;
  float acc = 0.f;
  for (int i = 0; i < F; ++i) acc = fmaf(fr[i], W[(P1 + i) * kH1 + cc], acc);
  out[(size_t)h * 128 + c] = acc;
}

}  // namespace

bool prb_fused_rollout_supported(prb_rollout r, prb_agent a, prb_vecenv env) {
  return env->kind == PRB_KIND_STOCK && a->hidden.size() == 2 && a->hidden[0] == kH1 && a->hidden[1] == kH2 &&
         env->A <= 31 && 1 + env->A <= (size_t)kXW && r->obs_mode == 1;
}

// worker_collect for the stock VecEnv as one fused launch (plus the tiny
// shared-layer kernel).  Host tracks the uniform t / done schedule.
void prb_fused_rollout_launch(prb_rollout r, prb_agent a, prb_vecenv env, uint64_t seed, std::vector<int32_t>& rows) {
  prb_ctx_s* ctx = r->ctx;
  cudaStream_t s = ctx->stream;
  const size_t N = r->N, H = r->H;
  const int K = env->market->K;
  prb_market_s* m = env->market;
  // the uniform t / done schedule of this rollout (stock_env.hpp:99-101,168)
  std::vector<int32_t> tseq(H + 1);
  std::vector<uint8_t> dseq(H);
  size_t t = env->t, sc = env->step_count;
  const int ep_len0 = (int)sc;
  for (size_t h = 0; h < H; ++h) {
    PRB_REQUIRE(t + 1 < m->T, PRB_ERR_USAGE, "stock_env_step: no next timestamp at t=" + std::to_string(t));
    tseq[h] = (int32_t)t;
    rows[h] = (int32_t)t;
    const size_t t1 = t + 1;
    const bool done = (t1 + 1 >= m->T) || (t1 >= env->end);
    dseq[h] = done ? 1 : 0;
    t = done ? env->start : t1;
    sc = done ? 0 : sc + 1;
  }
  tseq[H] = (int32_t)t;
  // small schedule + shared-layer buffers in the context scratch
  const size_t bytes_sl = (H + 1) * 128 * sizeof(float);
  const size_t bytes_t = ((H + 1) * sizeof(int32_t) + 15) & ~size_t(15);
  const size_t bytes_d = (H + 15) & ~size_t(15);
  char* scratch = static_cast<char*>(ctx->device_scratch(bytes_sl + bytes_t + bytes_d));
  float* d_sl = reinterpret_cast<float*>(scratch);
  int32_t* d_t = reinterpret_cast<int32_t*>(scratch + bytes_sl);
  uint8_t* d_d = reinterpret_cast<uint8_t*>(scratch + bytes_sl + bytes_t);
  int32_t* h_pin = static_cast<int32_t*>(ctx->pinned_staging(bytes_t + bytes_d));
  std::copy(tseq.begin(), tseq.end(), h_pin);
  std::copy(dseq.begin(), dseq.end(), reinterpret_cast<uint8_t*>(reinterpret_cast<char*>(h_pin) + bytes_t));
  PRB_CUDA(cudaMemcpyAsync(d_t, h_pin, bytes_t + bytes_d, cudaMemcpyHostToDevice, s));
  const int P1 = 1 + K, F = 5 * K;
  {
    ProfScope prof(ctx, kProfRollout);
    shared_layer1_kernel<<<(unsigned)(H + 1), 128, 0, s>>>(a->d_params.p, (int)a->aoff[0], (int)a->coff[0], P1, F,
                                                           env->d_feat.p, d_t, d_sl);
    FusedArgs f{};
    f.params = a->d_params.p;
    f.a_w1 = (int)a->aoff[0];
    f.a_w2 = (int)a->aoff[1];
    f.a_w3 = (int)a->aoff[2];
    f.c_w1 = (int)a->coff[0];
    f.c_w2 = (int)a->coff[1];
    f.c_w3 = (int)a->coff[2];
    f.log_std = (int)a->Pa;
    f.S = (int)env->S;
    f.K = K;
    f.shared_l1 = d_sl;
    f.t_seq = d_t;
    f.done_seq = d_d;
    f.close_tk = m->d_close_tk.p;
    f.feat = env->d_feat.p;
    f.cap = env->cfg.initial_capital;
    f.max_trade = env->cfg.max_trade_shares;
    f.cost = env->cfg.cost_rate;
    f.N = (int)N;
    f.H = (int)H;
    f.start = (int)env->start;
    f.ep_len0 = ep_len0;
    f.seed = seed;
    f.balance = env->d_balance.p;
    f.shares = env->d_shares.p;
    f.ep_return = env->d_ep_return.p;
    f.obs_out = env->d_obs.p;
    f.b_obs = r->d_obs.p;
    f.b_act = r->d_act.p;
    f.b_logp = r->d_logp.p;
    f.b_val = r->d_val.p;
    f.b_rew = r->d_rew.p;
    f.b_done = r->d_done.p;
    f.b_boot = r->d_boot.p;
    // tcgen05 bf16 MLP (rollout_tc.cu).  Its rare exact-division redo rebuilds the step's start
    // shares from the fp32 compact obs row, so every reachable share count must be an exact
    // float: at most max_trade_shares bought per step for at most end - start steps of an
    // episode (stock_env.hpp:91-97, :165-170) must stay below 2^24.
    const bool shares_exact_f32 =
        env->cfg.max_trade_shares * (double)(env->end - env->start + 1) < 16777216.0;
    if (r->mode == 2 && stock_rollout_tc_supported(K) && shares_exact_f32) {
      TcRolloutArgs ta{};
      ta.params = f.params;
      ta.a_w1 = f.a_w1; ta.a_w2 = f.a_w2; ta.a_w3 = f.a_w3;
      ta.c_w1 = f.c_w1; ta.c_w2 = f.c_w2; ta.c_w3 = f.c_w3;
      ta.log_std = f.log_std;
      ta.S = f.S; ta.K = f.K;
      ta.shared_l1 = f.shared_l1; ta.t_seq = f.t_seq; ta.done_seq = f.done_seq;
      ta.close_tk = f.close_tk; ta.feat = f.feat;
      ta.cap = f.cap; ta.max_trade = f.max_trade; ta.cost = f.cost;
      ta.mt_f32 = (f.max_trade == floor(f.max_trade) && f.max_trade >= 0.0 && f.max_trade < 4194304.0) ? 1 : 0;
      ta.force_redo = debug_option(PRB_OPT_TC_FORCE_REDO) ? 1 : 0;  // tests: the rare redo path every step
      ta.N = f.N; ta.H = f.H; ta.seed = f.seed;
      ta.balance = f.balance; ta.shares = f.shares; ta.ep_return = f.ep_return; ta.obs_out = f.obs_out;
      ta.b_obs = f.b_obs; ta.b_act = f.b_act; ta.b_logp = f.b_logp; ta.b_val = f.b_val; ta.b_rew = f.b_rew;
      ta.b_done = f.b_done; ta.b_boot = f.b_boot;
      const char* trace_path = debug_env("PRB_TC_TRACE");  // debug: clock64 phase trace of CTA 0
      DevBuf<unsigned long long> d_trace;
      if (trace_path) {
        // [kTcTraceLen] clock64 marks of CTA 0, then per CTA (smid, start, end) globaltimer stamps
        d_trace.alloc(kTcTraceLen + 3 * (size_t)((N + 127) / 128));
        PRB_CUDA(cudaMemsetAsync(d_trace.p, 0, d_trace.bytes(), s));
        ta.trace = d_trace.p;
      }
      launch_stock_rollout_tc(ta, s);
      if (trace_path) {
        std::vector<unsigned long long> hbuf(d_trace.n);
        PRB_CUDA(cudaMemcpyAsync(hbuf.data(), d_trace.p, d_trace.bytes(), cudaMemcpyDeviceToHost, s));
        PRB_CUDA(cudaStreamSynchronize(s));
        if (FILE* f = fopen(trace_path, "wb")) {
          fwrite(hbuf.data(), sizeof(unsigned long long), hbuf.size(), f);
          fclose(f);
        }
      }
    } else {  // fp32 SIMT MLP
      ensure_smem(stock_rollout_fused_kernel, sizeof(Smem));
      const unsigned grid = (unsigned)((N + kRows - 1) / kRows);
      stock_rollout_fused_kernel<<<grid, kThreads, sizeof(Smem), s>>>(f);
      PRB_CHECK_LAUNCH();
    }
  }
  env->t = t;
  env->step_count = sc;
}

// worker_collect of P pods' stock VecEnvs in ONE tcgen05 launch: each pod's
// uniform t / done schedule and shared first-layer term are prepared as for a single collect (its
// own buffers in the rollout), then pods x tiles CTAs run, each with its pod's weights, env state
// and rollout buffer.  Every pod: the tcgen05 stock path (64x64 nets, K in {1,2,3,30}), the same
// num_envs / horizon / K.
// whether P pods can be collected by ONE grouped tcgen05 launch (prb_tc_rollout_pods)
bool prb_tc_rollout_pods_supported(const prb_rollout* rs, const prb_agent* as, const prb_vecenv* es, size_t P) {
  const size_t N = rs[0]->N, H = rs[0]->H;
  if (es[0]->kind != PRB_KIND_STOCK) return false;
  const int K = es[0]->market->K;
  for (size_t p = 0; p < P; ++p) {
    prb_rollout r = rs[p];
    prb_vecenv env = es[p];
    if (env->kind != PRB_KIND_STOCK || r->N != N || r->H != H || env->N != N || env->market->K != K ||
        !prb_fused_rollout_supported(r, as[p], env) || !stock_rollout_tc_supported(K) ||
        !(env->cfg.max_trade_shares * (double)(env->end - env->start + 1) < 16777216.0))
      return false;
  }
  return true;
}

void prb_tc_rollout_pods(const prb_rollout* rs, const prb_agent* as, const prb_vecenv* es, size_t P,
                         const uint64_t* seeds) {
  prb_ctx_s* ctx = rs[0]->ctx;
  cudaStream_t s = ctx->stream;
  const size_t N = rs[0]->N, H = rs[0]->H;
  const int K = es[0]->market->K;
  std::vector<TcRolloutArgs> args(P);
  for (size_t p = 0; p < P; ++p) {
    prb_rollout r = rs[p];
    prb_agent a = as[p];
    prb_vecenv env = es[p];
    prb_market_s* m = env->market;
    PRB_REQUIRE(r->N == N && r->H == H && env->N == N && m->K == K && env->kind == PRB_KIND_STOCK &&
                    prb_fused_rollout_supported(r, a, env) && stock_rollout_tc_supported(K) &&
                    env->cfg.max_trade_shares * (double)(env->end - env->start + 1) < 16777216.0,
                PRB_ERR_USAGE, "worker_collect (pods): every pod needs the tcgen05 stock rollout and equal shapes");
    PRB_REQUIRE(env->was_reset, PRB_ERR_DIMENSION, "vec_step: sub-environments have no state (call reset first)");
    // this pod's schedule (stock_env.hpp:99-101,168) and shared-layer term in its own buffers
    std::vector<int32_t> tseq(H + 1);
    std::vector<uint8_t> dseq(H);
    size_t t = env->t, sc = env->step_count;
    for (size_t h = 0; h < H; ++h) {
      PRB_REQUIRE(t + 1 < m->T, PRB_ERR_USAGE, "stock_env_step: no next timestamp at t=" + std::to_string(t));
      tseq[h] = (int32_t)t;
      const size_t t1 = t + 1;
      const bool done = (t1 + 1 >= m->T) || (t1 >= env->end);
      dseq[h] = done ? 1 : 0;
      t = done ? env->start : t1;
      sc = done ? 0 : sc + 1;
    }
    tseq[H] = (int32_t)t;
    env->t = t;
    env->step_count = sc;
    r->d_sl.ensure((H + 1) * 128);
    r->d_tseq.ensure(H + 1);
    r->d_dseq.ensure(H);
    PRB_CUDA(cudaMemcpyAsync(r->d_tseq.p, tseq.data(), (H + 1) * sizeof(int32_t), cudaMemcpyHostToDevice, s));
    PRB_CUDA(cudaMemcpyAsync(r->d_dseq.p, dseq.data(), H, cudaMemcpyHostToDevice, s));
    PRB_CUDA(cudaMemcpyAsync(r->d_row.p, tseq.data(), H * sizeof(int32_t), cudaMemcpyHostToDevice, s));
    PRB_CUDA(cudaStreamSynchronize(s));  // tseq / dseq live on this stack frame
    {
      ProfScope prof(ctx, kProfRollout);
      shared_layer1_kernel<<<(unsigned)(H + 1), 128, 0, s>>>(a->d_params.p, (int)a->aoff[0], (int)a->coff[0], 1 + K,
                                                             5 * K, env->d_feat.p, r->d_tseq.p, r->d_sl.p);
    }
    PRB_CHECK_LAUNCH();
    TcRolloutArgs& ta = args[p];
    ta = TcRolloutArgs{};
    ta.params = a->d_params.p;
    ta.a_w1 = (int)a->aoff[0];
    ta.a_w2 = (int)a->aoff[1];
    ta.a_w3 = (int)a->aoff[2];
    ta.c_w1 = (int)a->coff[0];
    ta.c_w2 = (int)a->coff[1];
    ta.c_w3 = (int)a->coff[2];
    ta.log_std = (int)a->Pa;
    ta.S = (int)env->S;
    ta.K = K;
    ta.shared_l1 = r->d_sl.p;
    ta.t_seq = r->d_tseq.p;
    ta.done_seq = r->d_dseq.p;
    ta.close_tk = m->d_close_tk.p;
    ta.feat = env->d_feat.p;
    ta.cap = env->cfg.initial_capital;
    ta.max_trade = env->cfg.max_trade_shares;
    ta.cost = env->cfg.cost_rate;
    ta.mt_f32 = (ta.max_trade == floor(ta.max_trade) && ta.max_trade >= 0.0 && ta.max_trade < 4194304.0) ? 1 : 0;
    ta.N = (int)N;
    ta.H = (int)H;
    ta.seed = seeds[p];
    ta.balance = env->d_balance.p;
    ta.shares = env->d_shares.p;
    ta.ep_return = env->d_ep_return.p;
    ta.obs_out = env->d_obs.p;
    ta.b_obs = r->d_obs.p;
    ta.b_act = r->d_act.p;
    ta.b_logp = r->d_logp.p;
    ta.b_val = r->d_val.p;
    ta.b_rew = r->d_rew.p;
    ta.b_done = r->d_done.p;
    ta.b_boot = r->d_boot.p;
    r->d_feat = env->d_feat.p;
  }
  DevBuf<TcRolloutArgs> d_args;
  d_args.alloc(P);
  PRB_CUDA(cudaMemcpyAsync(d_args.p, args.data(), P * sizeof(TcRolloutArgs), cudaMemcpyHostToDevice, s));
  {
    ProfScope prof(ctx, kProfRollout);
    launch_stock_rollout_tc_group(d_args.p, (int)P, (int)N, K, s);
  }
  PRB_CUDA(cudaStreamSynchronize(s));  // d_args is released on return
}
