// rollout_tc.cu -- worker_collect (pod.hpp:95-132) for the stock VecEnv as one
// persistent kernel per rollout with the actor/critic MLP on the 5th-gen
// tensor cores (tcgen05.mma, bf16 operands in shared memory, fp32
// accumulators in TMEM).
//
// One CTA = 128 envs = one M=128 MMA tile = the 128 TMEM lanes; thread t owns
// env e0+t end to end (its TMEM lane, its obs row, its portfolio).  Per step:
//   A0 [128 x 32]  = bf16(balance/cap, shares)              (private obs; the
//                    150 shared features enter as the per-step layer-1 term)
//   L1: D[:,0:128] = A0 . W1p        -> +c_t +b1, tanh -> A1 bf16  (actor|critic)
//   L2: D[:,0:64]  = A1[:,0:64] . W2a ; D[:,64:128] = A1[:,64:128] . W2c -> tanh -> A1
//   L3: D[:,0:32]  = A1[:,0:64] . W3a ; D[:,32:48]  = A1[:,64:128] . W3c
//   Philox Gaussian sample + log-prob, stock_env_step in fp64 (thread-local,
//   reference operation order), coalesced compact rollout rows.
// Weights (bf16, 30 KB) and the portfolios stay on chip for all H steps;
// TMEM: 128 columns, reused by the three layers; 2 CTAs per SM overlap one
// CTA's fp64 env phase with the other's tensor-core layers.
#include <cuda_bf16.h>

#include <algorithm>

#include "prb_internal.h"
#include "rng.cuh"
#include "rollout_tc.h"
#include "tc.cuh"

namespace prb {
namespace {

constexpr int kM = 128;     // envs per CTA == MMA M == TMEM lanes
constexpr int kKX = 32;     // private obs width (1 + K <= 32)
constexpr int kMaxK = 31;
constexpr int kSP = kM + 1; // padded per-env column stride (bank-conflict free)
constexpr uint32_t kTmemCols = 128;
constexpr float kLogTwoPiF = 1.8378770664093454836f;

struct TcSmem {
  alignas(128) uint8_t w1[128 * kKX * 2];  // B [n=128][k=32]  W1 private rows, actor | critic
  alignas(128) uint8_t w2a[64 * 64 * 2];   // B [64][64]
  alignas(128) uint8_t w2c[64 * 64 * 2];
  alignas(128) uint8_t w3a[32 * 64 * 2];   // B [32][64]   (rows >= A zero)
  alignas(128) uint8_t w3c[16 * 64 * 2];   // B [16][64]   (row 0 = critic head)
  alignas(128) uint8_t a0[kM * kKX * 2];   // A [128][32]
  alignas(128) uint8_t a1[kM * 128 * 2];   // A [128][128]  h1, then h2
  float c1[128];
  float b2[128];
  float b3[32];
  float ls[32], sig[32];
  float b3c;
  float x0[kM];
  double p0[32], p1[32];
  int32_t sh[kMaxK][kSP];
  float act[kMaxK][kSP];
  uint64_t mbar;
  uint32_t tmem;
};

__device__ __forceinline__ double clamp_ref(double v, double lo, double hi) { return (v < lo) ? lo : ((hi < v) ? hi : v); }
__device__ __forceinline__ double min_ref(double a, double b) { return (b < a) ? b : a; }
__device__ __forceinline__ double max_ref(double a, double b) { return (a < b) ? b : a; }

__device__ __forceinline__ void st_bf16(uint8_t* base, uint32_t off, float v) {
  *reinterpret_cast<__nv_bfloat16*>(base + off) = __float2bfloat16_rn(v);
}

// 16 consecutive accumulator columns of this thread's row -> act -> bf16 into A1 (K-major)
template <bool TANH>
__device__ __forceinline__ void epilogue16(uint32_t taddr, const float* add, uint8_t* a1, int row, int c) {
  float v[16];
  tc::tmem_ld16(taddr, v);
  uint32_t pk[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    float x0 = v[2 * i] + add[c + 2 * i], x1 = v[2 * i + 1] + add[c + 2 * i + 1];
    if (TANH) {
      x0 = tc::tanh_fast(x0);
      x1 = tc::tanh_fast(x1);
    }
    pk[i] = tc::pack_bf16(x0, x1);
  }
  *reinterpret_cast<uint4*>(a1 + tc::kmajor_offset(row, c, 128)) = make_uint4(pk[0], pk[1], pk[2], pk[3]);
  *reinterpret_cast<uint4*>(a1 + tc::kmajor_offset(row, c + 8, 128)) = make_uint4(pk[4], pk[5], pk[6], pk[7]);
}

__global__ void __launch_bounds__(kM, 2) stock_rollout_tc_kernel(TcRolloutArgs a) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  TcSmem& s = *reinterpret_cast<TcSmem*>(smem_raw);
  const int tid = threadIdx.x, warp = tid >> 5;
  const int K = a.K, A = a.K, P1 = 1 + a.K, F = 5 * a.K;
  const size_t e0 = (size_t)blockIdx.x * kM;
  const int nloc = min(kM, a.N - (int)e0);
  const bool live = tid < nloc;
  const float* P = a.params;

  // ---- weights -> bf16 B operands (B[n][k] = W[k][n]), once per rollout ----
  for (int i = tid; i < 128 * kKX; i += kM) {
    const int n = i / kKX, k = i % kKX;
    float v = 0.f;
    if (k < P1) v = (n < 64) ? P[a.a_w1 + k * 64 + n] : P[a.c_w1 + k * 64 + (n - 64)];
    st_bf16(s.w1, tc::kmajor_offset(n, k, kKX), v);
  }
  for (int i = tid; i < 64 * 64; i += kM) {
    const int n = i / 64, k = i % 64;
    st_bf16(s.w2a, tc::kmajor_offset(n, k, 64), P[a.a_w2 + k * 64 + n]);
    st_bf16(s.w2c, tc::kmajor_offset(n, k, 64), P[a.c_w2 + k * 64 + n]);
  }
  for (int i = tid; i < 32 * 64; i += kM) {
    const int n = i / 64, k = i % 64;
    st_bf16(s.w3a, tc::kmajor_offset(n, k, 64), (n < A) ? P[a.a_w3 + k * A + n] : 0.f);
  }
  for (int i = tid; i < 16 * 64; i += kM) {
    const int n = i / 64, k = i % 64;
    st_bf16(s.w3c, tc::kmajor_offset(n, k, 64), (n == 0) ? P[a.c_w3 + k] : 0.f);
  }
  const float b1_mine = (tid < 64) ? P[a.a_w1 + a.S * 64 + tid] : P[a.c_w1 + a.S * 64 + tid - 64];
  s.b2[tid] = (tid < 64) ? P[a.a_w2 + 64 * 64 + tid] : P[a.c_w2 + 64 * 64 + tid - 64];
  if (tid < 32) {
    s.b3[tid] = (tid < A) ? P[a.a_w3 + 64 * A + tid] : 0.f;
    const float l = (tid < A) ? P[a.log_std + tid] : 0.f;
    s.ls[tid] = l;
    s.sig[tid] = expf(l);
  }
  if (tid == 0) s.b3c = P[a.c_w3 + 64];
  // ---- portfolio state: balance / episode return in registers, shares in smem ----
  double bal = live ? a.balance[e0 + tid] : a.cap;
  double ret = live ? a.ep_return[e0 + tid] : 0.0;
  for (int k = 0; k < K; ++k) s.sh[k][tid] = live ? a.shares[(size_t)k * a.N + e0 + tid] : 0;
  if (warp == 0) tc::tmem_alloc(&s.tmem, kTmemCols);
  if (tid == 0) tc::mbar_init(&s.mbar, 1);
  tc::fence_proxy_async();
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t tbase = s.tmem;
  const uint32_t tlane = tbase + ((uint32_t)(warp * 32) << 16);
  const uint32_t a0_addr = tc::smem_u32(s.a0), a1_addr = tc::smem_u32(s.a1);
  const uint32_t w1_addr = tc::smem_u32(s.w1), w2a_addr = tc::smem_u32(s.w2a), w2c_addr = tc::smem_u32(s.w2c);
  const uint32_t w3a_addr = tc::smem_u32(s.w3a), w3c_addr = tc::smem_u32(s.w3c);
  constexpr uint32_t ID_L1 = tc::idesc_bf16(128, 128), ID_L2 = tc::idesc_bf16(128, 64);
  constexpr uint32_t ID_L3A = tc::idesc_bf16(128, 32), ID_L3C = tc::idesc_bf16(128, 16);
  uint32_t phase = 0;
  const size_t row = e0 + tid;

  for (int h = 0; h <= a.H; ++h) {
    const int t = a.t_seq[h];
    s.c1[tid] = a.shared_l1[(size_t)h * 128 + tid] + b1_mine;
    if (tid < K) {
      s.p0[tid] = a.close_tk[(size_t)t * K + tid];
      if (h < a.H) s.p1[tid] = a.close_tk[(size_t)(t + 1) * K + tid];
    }
    // ---- A0 row: [balance/cap, shares] (stock_observation stock_env.hpp:115-121) ----
    const float xb = (float)__ddiv_rn(bal, a.cap);
    s.x0[tid] = xb;
    {
      float xv[kKX];
      xv[0] = xb;
#pragma unroll
      for (int k = 0; k < kMaxK; ++k) xv[1 + k] = (k < K) ? (float)s.sh[k][tid] : 0.f;
#pragma unroll
      for (int c = 0; c < kKX / 8; ++c) {
        const uint4 q = make_uint4(tc::pack_bf16(xv[8 * c], xv[8 * c + 1]), tc::pack_bf16(xv[8 * c + 2], xv[8 * c + 3]),
                                   tc::pack_bf16(xv[8 * c + 4], xv[8 * c + 5]), tc::pack_bf16(xv[8 * c + 6], xv[8 * c + 7]));
        *reinterpret_cast<uint4*>(s.a0 + tc::kmajor_offset(tid, 8 * c, kKX)) = q;
      }
    }
    tc::fence_proxy_async();
    tc::fence_before_sync();
    __syncthreads();
    if (tid == 0) {  // ---- L1: [128x32] . [32x128] ----
      tc::fence_after_sync();
#pragma unroll
      for (int j = 0; j < kKX / 16; ++j)
        tc::mma_bf16(tbase, tc::smem_desc(a0_addr + j * 256, 128, kKX * 16), tc::smem_desc(w1_addr + j * 256, 128, kKX * 16),
                     ID_L1, j > 0);
      tc::mma_commit(&s.mbar);
    }
    // overlap with the MMA: compact obs rows of step h / final VecEnv states
    if (h < a.H) {
      float* dst = a.b_obs + ((size_t)h * a.N + e0) * P1;
      for (int i = tid; i < nloc * P1; i += kM) {
        const int r = i / P1, c = i - (i / P1) * P1;
        dst[i] = (c == 0) ? s.x0[r] : (float)s.sh[c - 1][r];
      }
    } else {
      const float* fr = a.feat + (size_t)t * F;
      float* dst = a.obs_out + e0 * a.S;
      for (int i = tid; i < nloc * a.S; i += kM) {
        const int r = i / a.S, c = i - (i / a.S) * a.S;
        dst[i] = (c == 0) ? s.x0[r] : (c < P1 ? (float)s.sh[c - 1][r] : fr[c - P1]);
      }
    }
    tc::mbar_wait(&s.mbar, phase);
    phase ^= 1;
    tc::fence_after_sync();
    // ---- L1 epilogue: + shared term + b1, tanh -> A1 ----
#pragma unroll 1
    for (int c = 0; c < 128; c += 16) epilogue16<true>(tlane + c, s.c1, s.a1, tid, c);
    tc::fence_proxy_async();
    tc::fence_before_sync();
    __syncthreads();
    if (tid == 0) {  // ---- L2: actor / critic [128x64] . [64x64] ----
      tc::fence_after_sync();
#pragma unroll
      for (int j = 0; j < 4; ++j)
        tc::mma_bf16(tbase, tc::smem_desc(a1_addr + j * 256, 128, 2048), tc::smem_desc(w2a_addr + j * 256, 128, 1024),
                     ID_L2, j > 0);
#pragma unroll
      for (int j = 0; j < 4; ++j)
        tc::mma_bf16(tbase + 64, tc::smem_desc(a1_addr + 1024 + j * 256, 128, 2048),
                     tc::smem_desc(w2c_addr + j * 256, 128, 1024), ID_L2, j > 0);
      tc::mma_commit(&s.mbar);
    }
    tc::mbar_wait(&s.mbar, phase);
    phase ^= 1;
    tc::fence_after_sync();
#pragma unroll 1
    for (int c = 0; c < 128; c += 16) epilogue16<true>(tlane + c, s.b2, s.a1, tid, c);
    tc::fence_proxy_async();
    tc::fence_before_sync();
    __syncthreads();
    if (tid == 0) {  // ---- L3: actor head [128x64].[64x32], critic head [128x64].[64x16] ----
      tc::fence_after_sync();
#pragma unroll
      for (int j = 0; j < 4; ++j)
        tc::mma_bf16(tbase, tc::smem_desc(a1_addr + j * 256, 128, 2048), tc::smem_desc(w3a_addr + j * 256, 128, 1024),
                     ID_L3A, j > 0);
#pragma unroll
      for (int j = 0; j < 4; ++j)
        tc::mma_bf16(tbase + 32, tc::smem_desc(a1_addr + 1024 + j * 256, 128, 2048),
                     tc::smem_desc(w3c_addr + j * 256, 128, 1024), ID_L3C, j > 0);
      tc::mma_commit(&s.mbar);
    }
    tc::mbar_wait(&s.mbar, phase);
    phase ^= 1;
    tc::fence_after_sync();
    float mean[32], vcrit[16];
    tc::tmem_ld16(tlane + 0, mean);
    tc::tmem_ld16(tlane + 16, mean + 16);
    tc::tmem_ld16(tlane + 32, vcrit);
    tc::fence_before_sync();
#pragma unroll
    for (int d = 0; d < 32; ++d) mean[d] += s.b3[d];
    const float value = vcrit[0] + s.b3c;
    if (h == a.H) {  // bootstrap V(s_H) (pod.hpp:127-131)
      if (live) a.b_boot[row] = value;
      break;
    }
    // ---- sample a = mu + sigma * eps (Philox stream of policy_kernel), log-prob ----
    float lp = 0.f;
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      if (4 * q < A) {
        const Philox4 rr = philox4x32_10((uint32_t)a.seed, (uint32_t)(a.seed >> 32), (uint32_t)q, (uint32_t)row,
                                         (uint32_t)h, 0u);
        const float2 z0 = box_muller(rr.x, rr.y), z1 = box_muller(rr.z, rr.w);
        const float e4[4] = {z0.x, z0.y, z1.x, z1.y};
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int d = 4 * q + i;
          if (d < A) {
            const float act = mean[d] + s.sig[d] * e4[i];
            s.act[d][tid] = act;
            const float z = (act - mean[d]) / s.sig[d];
            lp += (-0.5f * kLogTwoPiF - s.ls[d]) - 0.5f * z * z;
          }
        }
      }
    }
    // ---- env step (stock_env_step stock_env.hpp:55-103), this thread's env, fp64 ----
    const int done = a.done_seq[h];
    float rew32 = 0.f;
    {
      double vb = bal;
      for (int k = 0; k < K; ++k) vb = __dadd_rn(vb, __dmul_rn((double)s.sh[k][tid], s.p0[k]));
      for (int k = 0; k < K; ++k) {
        const double d = trunc(__dmul_rn(clamp_ref((double)s.act[k][tid], -1.0, 1.0), a.max_trade));
        if (d < 0.0) {
          const int32_t held = s.sh[k][tid];
          const double qv = -min_ref(-d, (double)held);
          const double price = s.p0[k];
          const double cost = __dmul_rn(__dmul_rn(a.cost, fabs(qv)), price);
          bal = __dsub_rn(bal, __dadd_rn(__dmul_rn(qv, price), cost));
          s.sh[k][tid] = held + (int32_t)qv;
        }
      }
      const double cf = __dadd_rn(1.0, a.cost);
      for (int k = 0; k < K; ++k) {
        const double d = trunc(__dmul_rn(clamp_ref((double)s.act[k][tid], -1.0, 1.0), a.max_trade));
        if (d > 0.0) {
          const double price = s.p0[k];
          const double affordable = floor(__ddiv_rn(bal, __dmul_rn(price, cf)));
          const double qv = min_ref(d, max_ref(affordable, 0.0));
          const double cost = __dmul_rn(__dmul_rn(a.cost, fabs(qv)), price);
          bal = __dsub_rn(bal, __dadd_rn(__dmul_rn(qv, price), cost));
          s.sh[k][tid] += (int32_t)qv;
        }
      }
      double va = bal;
      for (int k = 0; k < K; ++k) va = __dadd_rn(va, __dmul_rn((double)s.sh[k][tid], s.p1[k]));
      const double rw = __dsub_rn(va, vb);
      rew32 = (float)rw;
      ret = __dadd_rn(ret, rw);
      if (done) {  // auto-reset (env.hpp:221-229, stock_env.hpp:158-163)
        bal = a.cap;
        ret = 0.0;
        for (int k = 0; k < K; ++k) s.sh[k][tid] = 0;
      }
    }
    __syncthreads();
    // ---- coalesced rollout writes of step h ----
    {
      const size_t slab = (size_t)h * a.N + e0;
      float* da = a.b_act + slab * A;
      for (int i = tid; i < nloc * A; i += kM) {
        const int r = i / A, k = i - (i / A) * A;
        da[i] = s.act[k][r];
      }
      if (live) {
        a.b_logp[slab + tid] = lp;
        a.b_val[slab + tid] = value;
        a.b_rew[slab + tid] = rew32;
        a.b_done[slab + tid] = (uint8_t)done;
      }
    }
  }
  // ---- portfolio state back to HBM ----
  __syncthreads();
  if (live) {
    a.balance[row] = bal;
    a.ep_return[row] = ret;
    for (int k = 0; k < K; ++k) a.shares[(size_t)k * a.N + row] = s.sh[k][tid];
  }
  tc::fence_before_sync();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc(tbase, kTmemCols);
}

}  // namespace

size_t stock_rollout_tc_smem() { return sizeof(TcSmem) + 1024; }

void launch_stock_rollout_tc(const TcRolloutArgs& a, cudaStream_t s) {
  static bool attr = false;
  if (!attr) {
    PRB_CUDA(cudaFuncSetAttribute(stock_rollout_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)stock_rollout_tc_smem()));
    attr = true;
  }
  const unsigned grid = (unsigned)((a.N + kM - 1) / kM);
  stock_rollout_tc_kernel<<<grid, kM, stock_rollout_tc_smem(), s>>>(a);
  PRB_CHECK_LAUNCH();
}

}  // namespace prb
