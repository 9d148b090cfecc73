// rollout_tc.cu -- worker_collect (pod.hpp:95-132) for the stock VecEnv as one
// persistent kernel per rollout with the actor/critic MLP on the 5th-gen
// tensor cores (tcgen05.mma, bf16 operands in shared memory, fp32
// accumulators in TMEM).
//
// One CTA = 128 envs = one M=128 MMA tile = the 128 TMEM lanes; thread t owns
// env e0+t end to end: its TMEM lane, its obs row, its portfolio (fp64
// balance / return and int32 shares in REGISTERS, K is a template constant).
// Per step (D = the CTA's 128 TMEM columns, X = one 16 KB bf16 operand tile):
//   X  <- bf16(balance/cap, shares)               [128 x 32]  private obs
//   L1 : D[0:128]  = X . W1p          (actor | critic; the 150 shared
//                                      features enter as the per-step term c_t)
//   X  <- tanh(D[0:64] + c_t)          actor h1      L2a: D[0:64]   = X . W2a
//   X  <- tanh(D[64:128] + c_t)        critic h1     L2c: D[64:128] = X . W2c
//   X  <- tanh(D[0:64] + b2)           actor h2      L3a: D[0:32]   = X . W3a (issued, not awaited)
//   value = tanh(D[64:128] + b2) . w3c + b3c   critic head in fp32 registers while L3a runs
//   Philox Gaussian sample + log-prob, stock_env_step in fp64 (thread-local,
//   reference operation order), rollout rows staged through X and written
//   warp-per-row (coalesced).
// One operand tile reused five times keeps shared memory at ~49 KB/CTA and
// TMEM at 128 columns/CTA, so 4 CTAs (512 envs) are resident per SM: the
// 65,536-env configs[1] VecEnv (512 tiles) runs as a single wave, and while one
// CTA waits on its tensor-core layer the others run epilogues / env steps.
#include <cuda_bf16.h>

#include <algorithm>

#include "prb_internal.h"
#include "rng.cuh"
#include "stock_env.cuh"
#include "rollout_tc.h"
#include "tc.cuh"

namespace prb {
namespace {

constexpr int kM = 128;     // envs per CTA == MMA M == TMEM lanes
constexpr int kKX = 32;     // private obs width (1 + K <= 32)
constexpr uint32_t kTmemCols = 128;
constexpr float kLogTwoPiF = 1.8378770664093454836f;
constexpr uint32_t kXLo = 8192;  // byte offset of the low-half private obs tile inside X
constexpr int kSLD = 31;    // fp32 staging row stride (odd: conflict-free both ways)

struct TcSmem {
  alignas(128) uint8_t w1[128 * kKX * 2];  // B [n=128][k=32]  W1 private rows, actor | critic
  alignas(128) uint8_t w2a[64 * 64 * 2];   // B [64][64]
  alignas(128) uint8_t w2c[64 * 64 * 2];
  alignas(128) uint8_t w3a[32 * 64 * 2];   // B [32][64]   (rows >= A zero)
  alignas(16) float w3c[64];               // critic head weights (fp32, SIMT dot product)
  alignas(128) uint8_t x[kM * 64 * 2];     // A tile: [128][32] obs, [128][64] h, fp32 [128][31] staging
  alignas(16) float c1[128];
  alignas(16) float b2[128];
  float b3[32];
  float sig[32], isig[32];
  float b3c, lpc;
  double p0[32], p1[32];
  stock::BuyPrice bp[32];
  uint64_t mbar;
  uint32_t tmem;
};

__device__ __forceinline__ double clamp_ref(double v, double lo, double hi) { return (v < lo) ? lo : ((hi < v) ? hi : v); }
__device__ __forceinline__ double min_ref(double a, double b) { return (b < a) ? b : a; }
__device__ __forceinline__ double max_ref(double a, double b) { return (a < b) ? b : a; }

__device__ __forceinline__ void st_bf16(uint8_t* base, uint32_t off, float v) {
  *reinterpret_cast<__nv_bfloat16*>(base + off) = __float2bfloat16_rn(v);
}

// 64 accumulator columns [col, col+64) of this thread's row -> tanh(. + add) -> bf16 X [128][64]
__device__ __forceinline__ void epilogue64(uint32_t tlane, int col, const float* add, uint8_t* x, int row) {
#pragma unroll 1
  for (int c = 0; c < 64; c += 16) {
    float v[16];
    tc::tmem_ld16(tlane + col + c, v);
    uint32_t pk[8];
    const float4* add4 = reinterpret_cast<const float4*>(add + col + c);  // 16-byte aligned (TcSmem)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const float4 b = add4[j];
      float z0 = v[4 * j], z1 = v[4 * j + 1], z2 = v[4 * j + 2], z3 = v[4 * j + 3];
      tc::add2(z0, z1, b.x, b.y);
      tc::add2(z2, z3, b.z, b.w);
      pk[2 * j] = tc::pack_bf16(tc::tanh_fast(z0), tc::tanh_fast(z1));
      pk[2 * j + 1] = tc::pack_bf16(tc::tanh_fast(z2), tc::tanh_fast(z3));
    }
    *reinterpret_cast<uint4*>(x + tc::arow_offset(row, c)) = make_uint4(pk[0], pk[1], pk[2], pk[3]);
    *reinterpret_cast<uint4*>(x + tc::arow_offset(row, c + 8)) = make_uint4(pk[4], pk[5], pk[6], pk[7]);
  }
}

// X written by the threads -> visible to the tensor core; all TMEM reads done.
__device__ __forceinline__ void publish_operand() {
  tc::fence_proxy_async();
  tc::fence_before_sync();
  __syncthreads();
}

// thread 0: D[d_col..] (+)= X[128 x 16*ksteps] . B ; commit; everyone waits.  X is in the
// row-interleaved layout (tc::arow_offset: K-step j at +j*4096, LBO 2048, SBO 128); with
// x_lo != 0 a second A tile at x_lo (the low bf16 halves of the same inputs) is accumulated
// against the same B, so the product sees X_hi + X_lo (~16 significant bits) instead of bf16(X).
__device__ __forceinline__ void mma_wait(uint64_t* mbar, uint32_t& phase) {
  tc::mbar_wait(mbar, phase);
  phase ^= 1;
  tc::fence_after_sync();
}

__device__ __forceinline__ void mma_layer(uint32_t tbase, uint32_t d_col, uint32_t x_addr, uint32_t b_addr,
                                          uint32_t b_sbo, int ksteps, uint32_t idesc, uint64_t* mbar,
                                          uint32_t& phase, uint32_t x_lo = 0, bool wait = true) {
  if (threadIdx.x == 0) {
    tc::fence_after_sync();
    for (int j = 0; j < ksteps; ++j)
      tc::mma_bf16(tbase + d_col, tc::smem_desc(x_addr + j * 4096, 2048, 128),
                   tc::smem_desc(b_addr + j * 256, 128, b_sbo), idesc, j > 0);
    if (x_lo)
      for (int j = 0; j < ksteps; ++j)
        tc::mma_bf16(tbase + d_col, tc::smem_desc(x_lo + j * 4096, 2048, 128),
                     tc::smem_desc(b_addr + j * 256, 128, b_sbo), idesc, 1);
    tc::mma_commit(mbar);
  }
  if (wait) mma_wait(mbar, phase);
}

// Copy of a staged tile that is already the contiguous [rows][cols] image of its HBM span (this
// CTA's rows are consecutive): 16-byte streaming stores (the rollout buffer is not re-read
// before the PPO update), scalar tail.  dst must be 16-byte aligned.
__device__ __forceinline__ void store_tile(float* __restrict__ dst, const float* stage, int nfl) {
  const int n4 = nfl >> 2;
  const float4* s4 = reinterpret_cast<const float4*>(stage);
  float4* d4 = reinterpret_cast<float4*>(dst);
  for (int i = threadIdx.x; i < n4; i += kM) __stcs(d4 + i, s4[i]);
  for (int i = (n4 << 2) + threadIdx.x; i < nfl; i += kM) __stcs(dst + i, stage[i]);
}

// store_tile for the action tile, then each thread turns the float4 it copied into the desired
// quantities (stock::desired_qty_f32) in place: conflict-free 16-byte shared accesses.
__device__ __forceinline__ void store_tile_desired(float* __restrict__ dst, float* stage, int nfl, float mt,
                                                   int32_t mti) {
  const int n4 = nfl >> 2;
  float4* s4 = reinterpret_cast<float4*>(stage);
  float4* d4 = reinterpret_cast<float4*>(dst);
  for (int i = threadIdx.x; i < n4; i += kM) {
    const float4 v = s4[i];
    __stcs(d4 + i, v);
    s4[i] = make_float4(__int_as_float(stock::desired_qty_f32(v.x, mt, mti)),
                        __int_as_float(stock::desired_qty_f32(v.y, mt, mti)),
                        __int_as_float(stock::desired_qty_f32(v.z, mt, mti)),
                        __int_as_float(stock::desired_qty_f32(v.w, mt, mti)));
  }
  for (int i = (n4 << 2) + threadIdx.x; i < nfl; i += kM) {
    const float v = stage[i];
    __stcs(dst + i, v);
    stage[i] = __int_as_float(stock::desired_qty_f32(v, mt, mti));
  }
}

// int32 -> double, exact either way: the XU conversion (1 issue slot, quarter-rate pipe) or the
// biased DADD (3 issue slots on the FMA/ALU pipes); PRB_TC_I2D_EXACT selects the latter.
__device__ __forceinline__ double to_f64(int32_t i) {
#ifdef PRB_TC_I2D_EXACT
  return stock::i2d_exact(i);
#else
  return (double)i;
#endif
}

// Desired quantities k, k+1 (k even) of this thread's staged row, re-read from shared memory on
// every use (volatile asm: the 30 values are not kept live next to the 30 share counts; no memory
// clobber, so the shared price loads around it can still be merged -- volatile asm keeps its
// order relative to the __syncthreads that publish the staged row).  The
// even stride 30 reads both with one 8-byte load, conflict-free per half-warp.
template <int SA>
__device__ __forceinline__ void desired_pair(const float* row, int k, int32_t& d0, int32_t& d1) {
  if constexpr (SA % 2 == 0) {
    asm volatile("ld.shared.v2.s32 {%0, %1}, [%2];" : "=r"(d0), "=r"(d1) : "r"(tc::smem_u32(row + k)));
  } else {
    asm volatile("ld.shared.s32 %0, [%1];" : "=r"(d0) : "r"(tc::smem_u32(row + k)));
    asm volatile("ld.shared.s32 %0, [%1];" : "=r"(d1) : "r"(tc::smem_u32(row + k + 1)));
  }
}

// Warp-per-row copy of the staged [rows][kSLD] fp32 tile to a contiguous [rows][cols] span.
__device__ __forceinline__ void store_rows(float* __restrict__ dst, const float* stage, int cols, int nrows,
                                           int sld = kSLD) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int r = warp; r < nrows; r += kM / 32)
    if (lane < cols) dst[(size_t)r * cols + lane] = stage[r * sld + lane];
}

template <int K, bool kTrace, typename Args>
__device__ __forceinline__ void rollout_tile(const Args& a, const int tile) {
  static_assert(K >= 1 && K <= 30, "private obs row and staging must fit 31 columns");
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  TcSmem& s = *reinterpret_cast<TcSmem*>(smem_raw);
  constexpr int A = K, P1 = 1 + K, F = 5 * K;
  // Staging strides: obs rows at kSLD (= P1 when K = 30: the staged tile is the contiguous image
  // of the CTA's obs rows), action rows at A when K = 30 (contiguous too; the 2-way bank
  // conflicts of stride 30 cost less than a row-by-row copy), else kSLD.
  constexpr int SA = (K == 30) ? A : kSLD;
  constexpr bool kTileObs = (P1 == kSLD), kTileAct = (SA == A);
  const bool vec_ok = (a.N & 3) == 0;  // 16-byte aligned spans of both tiles
  const int tid = threadIdx.x, warp = tid >> 5;
  const size_t e0 = (size_t)tile * kM;
  const int nloc = min(kM, a.N - (int)e0);
  const bool live = tid < nloc;
  const float* P = a.params;
  float* stage = reinterpret_cast<float*>(s.x);

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
  if (tid < 64) s.w3c[tid] = P[a.c_w3 + tid];
  const float b1_mine = (tid < 64) ? P[a.a_w1 + a.S * 64 + tid] : P[a.c_w1 + a.S * 64 + tid - 64];
  s.b2[tid] = (tid < 64) ? P[a.a_w2 + 64 * 64 + tid] : P[a.c_w2 + 64 * 64 + tid - 64];
  if (tid < 32) {
    s.b3[tid] = (tid < A) ? P[a.a_w3 + 64 * A + tid] : 0.f;
    const float l = (tid < A) ? P[a.log_std + tid] : 0.f;
    s.sig[tid] = expf(l);
    s.isig[tid] = expf(-l);
  }
  if (tid == 0) {
    s.b3c = P[a.c_w3 + 64];
    float c = 0.f;  // sum_d (-0.5 ln 2pi - log_std_d): the state-independent part of log pi
    for (int d = 0; d < A; ++d) c += -0.5f * kLogTwoPiF - P[a.log_std + d];
    s.lpc = c;
  }
  // ---- portfolio state in registers ----
  double bal = live ? a.balance[e0 + tid] : a.cap;
  double ret = live ? a.ep_return[e0 + tid] : 0.0;
  int32_t sh[K];
#pragma unroll
  for (int k = 0; k < K; ++k) sh[k] = live ? a.shares[(size_t)k * a.N + e0 + tid] : 0;
  if (warp == 0) tc::tmem_alloc(&s.tmem, kTmemCols);
  if (tid == 0) tc::mbar_init(&s.mbar, 1);
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t tbase = s.tmem;
  const uint32_t tlane = tbase + ((uint32_t)(warp * 32) << 16);
  const uint32_t x_addr = tc::smem_u32(s.x);
  const uint32_t w1_addr = tc::smem_u32(s.w1), w2a_addr = tc::smem_u32(s.w2a), w2c_addr = tc::smem_u32(s.w2c);
  const uint32_t w3a_addr = tc::smem_u32(s.w3a);
  constexpr uint32_t ID_L1 = tc::idesc_bf16(128, 128), ID_L2 = tc::idesc_bf16(128, 64);
  constexpr uint32_t ID_L3A = tc::idesc_bf16(128, 32);
  uint32_t phase = 0;
  const size_t row = e0 + tid;
  tc::Tracer<kTcTraceLen, kTrace> tr;
  if (a.trace && tile == 0 && tid == 0) tr.p = a.trace;
  // value_before of the first step (stock_env.hpp:68); later steps carry value_after
  double vb = bal;
  {
    const int t0 = a.t_seq[0];
#pragma unroll
    for (int k = 0; k < K; ++k) vb = __dadd_rn(vb, __dmul_rn((double)sh[k], a.close_tk[(size_t)t0 * K + k]));
  }

  for (int h = 0; h <= a.H; ++h) {
    const int t = a.t_seq[h];
    __syncthreads();  // previous step's staging reads of X are done
    tr.mark();
    s.c1[tid] = a.shared_l1[(size_t)h * 128 + tid] + b1_mine;
    if (tid < K) {
      const double p0 = a.close_tk[(size_t)t * K + tid];
      s.p0[tid] = p0;
      s.bp[tid] = stock::buy_price(p0, a.cost);
      if (h < a.H) s.p1[tid] = a.close_tk[(size_t)(t + 1) * K + tid];
    }
    // ---- X <- [balance/cap, shares] (stock_observation stock_env.hpp:115-121) ----
    const float x0 = (float)__ddiv_rn(bal, a.cap);
    {  // hi / lo bf16 halves: raw share counts need more than bf16's 8 bits (integers < 2^16 exact)
      float xv[kKX];
      xv[0] = x0;
#pragma unroll
      for (int k = 0; k < kKX - 1; ++k) xv[1 + k] = (k < K) ? (float)sh[k] : 0.f;
#pragma unroll
      for (int c = 0; c < kKX / 8; ++c) {
        uint32_t hi[4], lo[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          hi[i] = tc::pack_bf16(xv[8 * c + 2 * i], xv[8 * c + 2 * i + 1]);
          lo[i] = tc::pack_bf16(xv[8 * c + 2 * i] - __uint_as_float(hi[i] << 16),
                                xv[8 * c + 2 * i + 1] - __uint_as_float(hi[i] & 0xFFFF0000u));
        }
        *reinterpret_cast<uint4*>(s.x + tc::arow_offset(tid, 8 * c)) = make_uint4(hi[0], hi[1], hi[2], hi[3]);
        *reinterpret_cast<uint4*>(s.x + kXLo + tc::arow_offset(tid, 8 * c)) = make_uint4(lo[0], lo[1], lo[2], lo[3]);
      }
    }
    tr.mark();
    publish_operand();
    mma_layer(tbase, 0, x_addr, w1_addr, kKX * 16, kKX / 16, ID_L1, &s.mbar, phase, x_addr + kXLo);  // L1
    tr.mark();
    epilogue64(tlane, 0, s.c1, s.x, tid);                                                          // actor h1
    tr.mark();
    publish_operand();
    mma_layer(tbase, 0, x_addr, w2a_addr, 1024, 4, ID_L2, &s.mbar, phase);                   // L2a
    tr.mark();
    epilogue64(tlane, 64, s.c1, s.x, tid);                                                         // critic h1
    tr.mark();
    publish_operand();
    mma_layer(tbase, 64, x_addr, w2c_addr, 1024, 4, ID_L2, &s.mbar, phase);                  // L2c
    tr.mark();
    epilogue64(tlane, 0, s.b2, s.x, tid);                                                          // actor h2
    tr.mark();
    publish_operand();
    mma_layer(tbase, 0, x_addr, w3a_addr, 1024, 4, ID_L3A, &s.mbar, phase, 0, false);  // L3a: issue only
    tr.mark();
    // critic head while L3a runs: value = tanh(D[64:128] + b2) . w3c + b3c in fp32 (the 64-wide dot
    // product is cheaper on the FMA pipe than a round trip through X and a 5th MMA; L3a writes
    // D[0:32] only)
    float value;
    {
      float acc = 0.f;
#pragma unroll 1
      for (int c = 0; c < 64; c += 16) {
        float v[16];
        tc::tmem_ld16(tlane + 64 + c, v);
        const float4* b4 = reinterpret_cast<const float4*>(s.b2 + 64 + c);
        const float4* w4 = reinterpret_cast<const float4*>(s.w3c + c);
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const float4 b = b4[j], w = w4[j];
          float z0 = v[4 * j], z1 = v[4 * j + 1], z2 = v[4 * j + 2], z3 = v[4 * j + 3];
          tc::add2(z0, z1, b.x, b.y);
          tc::add2(z2, z3, b.z, b.w);
          acc = fmaf(tc::tanh_fast(z0), w.x, acc);
          acc = fmaf(tc::tanh_fast(z1), w.y, acc);
          acc = fmaf(tc::tanh_fast(z2), w.z, acc);
          acc = fmaf(tc::tanh_fast(z3), w.w, acc);
        }
      }
      value = acc + s.b3c;
    }
    tr.mark();
    mma_wait(&s.mbar, phase);  // L3a done: the actor head is in D[0:32]
    tr.mark();
    // no barrier needed before staging into X: L3a (X's last reader) is complete for every
    // thread that has passed its own mbarrier wait, and the next MMA is behind publish_operand
    if (h == a.H) {  // bootstrap V(s_H) (pod.hpp:127-131) and the VecEnv's final states
      tc::fence_before_sync();
      if (live) a.b_boot[row] = value;
      stage[tid * kSLD] = x0;
#pragma unroll
      for (int k = 0; k < K; ++k) stage[tid * kSLD + 1 + k] = (float)sh[k];
      __syncthreads();
      const float* fr = a.feat + (size_t)t * F;
      const int lane = tid & 31;
      for (int r = warp; r < nloc; r += kM / 32) {
        float* dst = a.obs_out + (e0 + r) * a.S;
        if (lane < P1) dst[lane] = stage[r * kSLD + lane];
        for (int c = lane; c < F; c += 32) dst[P1 + c] = fr[c];
      }
      break;
    }
    // ---- compact obs rows of step h ----
    stage[tid * kSLD] = x0;
#pragma unroll
    for (int k = 0; k < K; ++k) stage[tid * kSLD + 1 + k] = (float)sh[k];
    __syncthreads();
    if (kTileObs && vec_ok)
      store_tile(a.b_obs + ((size_t)h * a.N + e0) * P1, stage, nloc * P1);
    else
      store_rows(a.b_obs + ((size_t)h * a.N + e0) * P1, stage, P1, nloc);
    __syncthreads();
    tr.mark();
    // ---- a = mu + sigma * eps (Philox stream of policy_kernel), log-prob; actions staged ----
    float zz = 0.f;
#pragma unroll
    for (int half = 0; half < 2; ++half) {
      if (16 * half < A) {
        float mean[16];
        tc::tmem_ld16(tlane + 16 * half, mean);
#pragma unroll
        for (int qq = 0; qq < 4; ++qq) {
          const int q = 4 * half + qq;
          if (4 * q < A) {
            const Philox4 rr = philox4x32_10((uint32_t)a.seed, (uint32_t)(a.seed >> 32), (uint32_t)q, (uint32_t)row,
                                             (uint32_t)h, 0u);
            const float2 z0 = box_muller(rr.x, rr.y), z1 = box_muller(rr.z, rr.w);
            const float e4[4] = {z0.x, z0.y, z1.x, z1.y};
#pragma unroll
            for (int i = 0; i < 4; ++i) {
              const int d = 4 * q + i;
              if (d < A) {
                const float m = mean[4 * qq + i] + s.b3[d];
                const float act = m + s.sig[d] * e4[i];
                zz += e4[i] * e4[i];  // z = (a - mu) / sigma is eps up to the rounding of a
                stage[tid * SA + d] = act;
              }
            }
          }
        }
      }
    }
    tc::fence_before_sync();
    const float lp = s.lpc - 0.5f * zz;
    __syncthreads();
    tr.mark();
    // desired_k = trunc(clamp(a_k, -1, 1) * max_trade) (stock_env.hpp:83-87) ONCE per step, as
    // int32 bit patterns written over the staged action tile: in the vectorised tile copy when it
    // applies (each thread converts the float4 it has just stored), else row by row.
    const bool tile_desired = kTileAct && vec_ok && a.mt_f32;
    if (tile_desired)
      store_tile_desired(a.b_act + ((size_t)h * a.N + e0) * A, stage, nloc * A, (float)a.max_trade,
                         (int32_t)a.max_trade);
    else if (kTileAct && vec_ok)
      store_tile(a.b_act + ((size_t)h * a.N + e0) * A, stage, nloc * A);
    else
      store_rows(a.b_act + ((size_t)h * a.N + e0) * A, stage, A, nloc, SA);
    tr.mark();
    // ---- env step (stock_env_step stock_env.hpp:55-103), this thread's env, fp64 ----
    // The desired quantities are re-read from this thread's staged row in each loop (8-byte
    // loads at the even stride 30: conflict-free per half-warp) instead of being kept live next
    // to the 30 share counts.  Sells run in integers except the cash arithmetic; buys use
    // stock::buy_qty_i32 (no fp64 division on the balance chain, stock_env.cuh); every trade is
    // branch-free (a zero-quantity trade leaves balance and shares bit-identical).
    __syncthreads();  // the act tile copy (and its in-place conversion) is complete
    float* my = stage + tid * SA;
    if (!tile_desired) {
      if (a.mt_f32) {
        const float mtf = (float)a.max_trade;
        const int32_t mti = (int32_t)a.max_trade;
#pragma unroll
        for (int k = 0; k < K; ++k) my[k] = __int_as_float(stock::desired_qty_f32(my[k], mtf, mti));
      } else {
#pragma unroll
        for (int k = 0; k < K; ++k)
          my[k] = __int_as_float((int32_t)trunc(__dmul_rn(clamp_ref((double)my[k], -1.0, 1.0), a.max_trade)));
      }
    }
    const int done = a.done_seq[h];
    const double bal_s = bal;  // for the rare redo below
    bool bad = a.force_redo != 0;  // a buy quantity outside stock::buy_qty_i32_spec's certificate
    auto sell = [&](int k, int32_t di) {  // sells first (:88-90): q = -min(-d, shares), exact in int32
      const int32_t qi = min(max(di, -sh[k]), 0);
      const double qv = to_f64(qi);
      const double price = s.p0[k];
      const double cost = __dmul_rn(__dmul_rn(a.cost, fabs(qv)), price);
      bal = __dsub_rn(bal, __dadd_rn(__dmul_rn(qv, price), cost));
      sh[k] += qi;
    };
    auto buy = [&](int k, int32_t di) {  // then buys, clipped to the affordable balance incl. cost (:91-97)
      const int32_t qi = stock::buy_qty_i32_spec(di, bal, s.bp[k], bad);
      const double qv = to_f64(qi);
      const double price = s.p0[k];
      const double cost = __dmul_rn(__dmul_rn(a.cost, qv), price);
      bal = __dsub_rn(bal, __dadd_rn(__dmul_rn(qv, price), cost));
      sh[k] += qi;
    };
#pragma unroll
    for (int k = 0; k < K; k += 2) {
      int32_t d0, d1;
      desired_pair<SA>(my, k, d0, d1);
      sell(k, d0);
      if (k + 1 < K) sell(k + 1, d1);
    }
#pragma unroll
    for (int k = 0; k < K; k += 2) {
      int32_t d0, d1;
      desired_pair<SA>(my, k, d0, d1);
      buy(k, d0);
      if (k + 1 < K) buy(k + 1, d1);
    }
    if (__any_sync(0xffffffffu, bad)) {
      // Some lane's quotient was within 2^-19 of an integer (or its cash <= 0): redo this step's
      // trades for the warp with the reference's division, from the shares at the start of the
      // step (this row of the compact obs tile written above) and bal_s.  The floats are the
      // exact share counts: the launcher routes here only when every reachable count is below
      // 2^24 (rollout_fused.cu).
      const float* orow = a.b_obs + ((size_t)h * a.N + row) * P1 + 1;
#pragma unroll
      for (int k = 0; k < K; ++k) sh[k] = live ? (int32_t)orow[k] : 0;
      bal = bal_s;
      const double cf = __dadd_rn(1.0, a.cost);
#pragma unroll
      for (int k = 0; k < K; ++k) {
        const int32_t di = __float_as_int(my[k]);
        if (di < 0) {
          const int32_t q = -min(-di, sh[k]);
          const double qv = (double)q;
          bal = __dsub_rn(bal, __dadd_rn(__dmul_rn(qv, s.p0[k]), __dmul_rn(__dmul_rn(a.cost, fabs(qv)), s.p0[k])));
          sh[k] += q;
        }
      }
#pragma unroll
      for (int k = 0; k < K; ++k) {
        const int32_t di = __float_as_int(my[k]);
        if (di > 0) {
          const double qv = stock::buy_qty((double)di, bal, __dmul_rn(s.p0[k], cf));
          bal = __dsub_rn(bal, __dadd_rn(__dmul_rn(qv, s.p0[k]), __dmul_rn(__dmul_rn(a.cost, qv), s.p0[k])));
          sh[k] += (int32_t)qv;
        }
      }
    }
    double va = bal;
#pragma unroll
    for (int k = 0; k < K; ++k) va = __dadd_rn(va, __dmul_rn(to_f64(sh[k]), s.p1[k]));
    const double rw = __dsub_rn(va, vb);
    ret = __dadd_rn(ret, rw);
    // next step's value_before: the same shares at close[t+1] plus the same balance is exactly
    // this step's value_after (same operands, same order); after an auto-reset it is
    // cap + sum(0 * close) = cap
    vb = done ? a.cap : va;
    tr.mark();
    if (done) {  // auto-reset (env.hpp:221-229, stock_env.hpp:158-163)
      bal = a.cap;
      ret = 0.0;
#pragma unroll
      for (int k = 0; k < K; ++k) sh[k] = 0;
    }
    if (live) {
      const size_t slab = (size_t)h * a.N + row;
      a.b_logp[slab] = lp;
      a.b_val[slab] = value;
      a.b_rew[slab] = (float)rw;
      a.b_done[slab] = (uint8_t)done;
    }
    tr.mark();
  }
  // ---- portfolio state back to HBM ----
  if (live) {
    a.balance[row] = bal;
    a.ep_return[row] = ret;
#pragma unroll
    for (int k = 0; k < K; ++k) a.shares[(size_t)k * a.N + row] = sh[k];
  }
  tc::fence_before_sync();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc(tbase, kTmemCols);
}

template <int K, bool kTrace>
__global__ void __launch_bounds__(kM, 4) stock_rollout_tc_kernel(TcRolloutArgs a) {
  rollout_tile<K, kTrace>(a, (int)blockIdx.x);
}

// P pods' collects in one launch: CTA b runs tile b % tiles of pod
// b / tiles with that pod's weights, env state and buffer (a grouped GEMM over the pods)
template <int K>
__global__ void __launch_bounds__(kM, 4) stock_rollout_tc_group_kernel(const TcRolloutArgs* __restrict__ group,
                                                                       int tiles) {
  rollout_tile<K, false>(group[blockIdx.x / tiles], (int)(blockIdx.x % tiles));
}

}  // namespace

size_t stock_rollout_tc_smem() { return sizeof(TcSmem); }

bool stock_rollout_tc_supported(int K) { return K == 30 || K == 3 || K == 2 || K == 1; }

void launch_stock_rollout_tc_group(const TcRolloutArgs* d_group, int pods, int N, int K, cudaStream_t s) {
  const int tiles = (N + kM - 1) / kM;
  const size_t smem = stock_rollout_tc_smem();
  switch (K) {
    case 30:
      ensure_smem(stock_rollout_tc_group_kernel<30>, smem);
      stock_rollout_tc_group_kernel<30><<<(unsigned)(pods * tiles), kM, smem, s>>>(d_group, tiles);
      break;
    case 3:
      ensure_smem(stock_rollout_tc_group_kernel<3>, smem);
      stock_rollout_tc_group_kernel<3><<<(unsigned)(pods * tiles), kM, smem, s>>>(d_group, tiles);
      break;
    default:
      fail(PRB_ERR_CONFIG, "grouped tcgen05 rollout: no instantiation for K=" + std::to_string(K));
  }
  PRB_CHECK_LAUNCH();
}

void launch_stock_rollout_tc(const TcRolloutArgs& a, cudaStream_t s) {
  const unsigned grid = (unsigned)((a.N + kM - 1) / kM);
  const size_t smem = stock_rollout_tc_smem();
#define PRB_TC_CASE(KK)                                                                                      \
  case KK: {                                                                                                 \
    ensure_smem(stock_rollout_tc_kernel<KK, false>, smem);                                                   \
    ensure_smem(stock_rollout_tc_kernel<KK, true>, smem);                                                    \
    if (a.trace)                                                                                             \
      stock_rollout_tc_kernel<KK, true><<<grid, kM, smem, s>>>(a);                                           \
    else                                                                                                     \
      stock_rollout_tc_kernel<KK, false><<<grid, kM, smem, s>>>(a);                                          \
    break;                                                                                                   \
  }
  switch (a.K) {
    PRB_TC_CASE(30)
    PRB_TC_CASE(3)
    PRB_TC_CASE(2)
    PRB_TC_CASE(1)
    default:
      fail(PRB_ERR_CONFIG, "tcgen05 rollout: no instantiation for K=" + std::to_string(a.K));
  }
#undef PRB_TC_CASE
  PRB_CHECK_LAUNCH();
}

}  // namespace prb
