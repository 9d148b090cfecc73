// ppo_tc.cu -- ppo_update (ppo.hpp:249-296) on the 5th-gen tensor cores, one thread-block
// cluster per learner.
//
// A learner's update is a chain of minibatch steps (gather_minibatch ppo.hpp:83-103 ->
// detail::ppo_loss_grads :116-188 -> adam_step nn.hpp:164-182).  Here the C = ceil(mb / 128)
// CTAs of one cluster run the whole chain (every epoch, every minibatch) in one launch, without
// grid-wide barriers, so several learners (pod.hpp:436-461) run at once,
// one cluster each.  Per step, CTA c of the cluster owns minibatch rows [128c, 128c + 128):
//
//   gather    X = [private features hi | rest | 1] per row as bf16 hi + lo pairs  [128 x 192]
//   L1        D = X_hi . W1 + X_lo . W1        (actor | critic: N = 128; b1 via the ones column)
//   L2        H1 = tanh(D);  D = H1_a . W2a,  D = H1_c . W2c        (+ b2 in the epilogue)
//   heads     H2 = tanh(D);  D = H2_a . W3a (N = 32),  D = H2_c . W3c (N = 16)
//   head grads (per row, fp32: log-prob, ratio, clipped surrogate with the tie rule of
//             ppo.hpp:146, value error)           -> d3 = [dmu / sigma-scaled | dV]
//   backward  d2 = (d3 . W3^T) o (1 - H2^2)  (actor by MMA, critic as an outer product)
//             d1 = (d2 . W2^T) o (1 - H1^2)
//   weight gradients, batch as the contraction dimension (both operands MN-major):
//             dW3^T = d3^T . H2,  dW2^T = d2^T . H1,  dW1^T = d1^T . X_hi   (fp32 in TMEM)
//   partials  TMEM -> this CTA's slab row (flat parameter order) + log_std / loss terms
//   cluster barrier; CTA c sums the C slab rows of its 1/C parameter slice in rank order,
//   evaluates its part of the finiteness gate (losses first, then gradients, the reference's
//   order), exchanges the gate over DSMEM; if every part passed, Adam on its slice (fp32 master
//   weights, adam_param's explicit roundings) and the slice's entries of the bf16 weight image;
//   cluster barrier; every CTA bulk-copies the image (72 KB) for the next step.
//
// Every matrix lives in shared memory once, in the "row-fast core form" of tc.cuh (8x8 bf16 core
// matrices, 8-row groups 128 B apart, 8-column chunks R*16 B apart), which is the K-major operand
// layout when its columns are the contraction dimension and the MN-major (transposed) layout when
// its rows are: the forward and backward read the same bytes with different descriptors.
// TMEM (512 columns): L1 [0,128) L2 [128,256) heads [256,304) -> dW3^T [0,128) dW2^T [128,256)
// dW1^T [256,448), with the backward accumulators d2a [256,320) and d1 [320,448) consumed before
// dW1^T is issued.  Precision: bf16 operands, fp32 accumulation and elementwise math; the
// inputs as hi + lo bf16 pairs (~16 significant bits) in the forward.
#include <cuda_bf16.h>

#include <algorithm>
#include <cmath>
#include <cstring>

#include "ppo_tc.h"
#include "prb_internal.h"
#include "rng.cuh"
#include "tc.cuh"

namespace prb {
namespace {

#ifndef PRB_TC_MN_LBO_IS_MN
#define PRB_TC_MN_LBO_IS_MN 0
#endif
// MN-major (no swizzle) descriptors: LBO = the core-matrix stride along K, SBO = along MN (the
// canonical ((8,m),(8,k)) : ((16 B, SBO), (16 B rows, LBO)) form; measured, profiles/tc_major_probe.py)
constexpr bool kMnLboIsMn = PRB_TC_MN_LBO_IS_MN;

constexpr int kRows = 128;
constexpr int kThreads = 256;
constexpr int kXC = 192;  // X columns
constexpr int kHC = 128;  // H1 / H2 / d1 / d2 / d3 columns (actor 0-63 | critic 64-127)
constexpr float kLogTwoPiF = 1.8378770664093454836f;

// shared-memory map (bytes from the 1024-aligned dynamic base)
constexpr uint32_t kOffXhi = 0;                        // X_hi   [128][192]            49152
constexpr uint32_t kOffRB = 49152;                     // X_lo [128][192] | BUF1 + BUF2
constexpr uint32_t kOffBuf1 = kOffRB;                  // d3 / d1 [128][128]          32768
constexpr uint32_t kOffBuf2 = kOffRB + 32768;          // d2 [128][128] (+ fp32 reduce scratch)
constexpr uint32_t kOffRC = kOffRB + 65536;            // W1 image [128 out][192] | H1 [128][128]
constexpr uint32_t kOffH2 = kOffRC + 49152;            // H2 [128][128]               32768
constexpr uint32_t kOffRE = kOffH2 + 32768;            // W2a, W2c [64][64], W3a [64][32], W3c [64][16]
constexpr uint32_t kOffW2a = kOffRE, kOffW2c = kOffRE + 8192, kOffW3a = kOffRE + 16384, kOffW3c = kOffRE + 20480;
constexpr uint32_t kOffF32 = kOffRE + 22528;           // fp32 block (image tail)        1040
constexpr uint32_t kOffRows = kOffF32 + 1040;          // per-row old_lp, adv, ret, dv [4][128] fp32
constexpr uint32_t kOffRidx = kOffRows + 2048;         // per-row buffer index [128] u32
constexpr uint32_t kSmemBytes = kOffRidx + 512;
// image (global) = W1 block | RE | fp32 block, the smem bytes [kOffRC, +49152) ++ [kOffRE, +23568)
constexpr uint32_t kImgW1 = 49152, kImgRest = 22528 + 1040;
static_assert(kImgW1 + kImgRest == (uint32_t)kPpoTcImgBytes, "image size");
// fp32 block (float index): b2 [0,128), b3a [128,160), b3c 160, log_std [164,196), w3c [196,260)
constexpr int kFb2 = 0, kFb3a = 128, kFb3c = 160, kFls = 164, kFw3c = 196;

// byte offset of element (r, c) of a [R][*] matrix in the row-fast core form
__host__ __device__ __forceinline__ uint32_t core_off(int r, int c, int R) {
  return (uint32_t)((c >> 3) * (R * 16) + (r >> 3) * 128 + (r & 7) * 16 + (c & 7) * 2);
}

// descriptors of an R-row matrix at `addr`: its columns as K (K-major) or its rows as K (MN-major)
__device__ __forceinline__ uint64_t desc_k(uint32_t addr, int R) { return tc::smem_desc(addr, R * 16, 128); }
__device__ __forceinline__ uint64_t desc_mn(uint32_t addr, int R) {
  return kMnLboIsMn ? tc::smem_desc(addr, R * 16, 128) : tc::smem_desc(addr, 128, R * 16);
}

// D (+)= A . B over `ksteps` K-steps of 16.  a_mn / b_mn: operand read MN-major (K = its rows).
__device__ __forceinline__ void mma_chain(uint32_t d_tmem, uint32_t a_addr, int a_rows, int a_mn, uint32_t b_addr,
                                          int b_rows, int b_mn, int ksteps, int N, bool accumulate) {
  const uint32_t idesc = tc::idesc_bf16_t(128, N, a_mn, b_mn);
  const uint32_t a_step = a_mn ? 256u : (uint32_t)a_rows * 32u;
  const uint32_t b_step = b_mn ? 256u : (uint32_t)b_rows * 32u;
  for (int j = 0; j < ksteps; ++j) {
    const uint64_t ad = a_mn ? desc_mn(a_addr + j * a_step, a_rows) : desc_k(a_addr + j * a_step, a_rows);
    const uint64_t bd = b_mn ? desc_mn(b_addr + j * b_step, b_rows) : desc_k(b_addr + j * b_step, b_rows);
    tc::mma_bf16(d_tmem, ad, bd, idesc, (accumulate || j > 0) ? 1u : 0u);
  }
}

__device__ __forceinline__ void cluster_arrive() { asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory"); }
__device__ __forceinline__ void cluster_wait() { asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory"); }
__device__ __forceinline__ void st_cluster_u32(uint32_t cluster_addr, uint32_t v) {
  asm volatile("st.shared::cluster.u32 [%0], %1;" ::"r"(cluster_addr), "r"(v) : "memory");
}

// Keyed balanced-Feistel bijection on [0, 2^bits), cycle-walked into [0, n) -- the same
// permutation the SIMT update draws (ppo.cu), so both paths see the same minibatches.
__device__ __forceinline__ uint32_t feistel(uint32_t x, uint32_t n, int bits, uint64_t key) {
  const int h = bits >> 1;
  const uint32_t mask = (h >= 32) ? 0xffffffffu : ((1u << h) - 1u);
  do {
    uint32_t L = x >> h, Rr = x & mask;
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const uint32_t f = (uint32_t)splitmix64_d(key + 0x9E3779B97F4A7C15ULL * (uint64_t)(r + 1) + Rr) & mask;
      const uint32_t nl = Rr, nr = L ^ f;
      L = nl;
      Rr = nr;
    }
    x = (L << h) | Rr;
  } while (x >= n);
  return x;
}

__device__ __forceinline__ uint32_t mb_index(const PpoTcArgs& a, const PpoTcChain& ch, int64_t step, uint32_t q) {
  const uint32_t epoch = (uint32_t)(step / a.nmb);
  const uint32_t pos = (uint32_t)(step % a.nmb) * (uint32_t)a.mb + q;
  if (ch.perm) return ch.perm[(size_t)epoch * a.n + pos];
  return feistel(pos, a.n, a.bits, derive_seed2(ch.seed, 0x50504fULL /*"PPO"*/, epoch));
}

// adam_step (nn.hpp:164-182) for one fp32 parameter, every rounding explicit (as ppo.cu)
__device__ __forceinline__ void adam_param(float b1, float b2, float omb1, float omb2, float lr, float eps, float ibc1,
                                           float ibc2, float g, float& m, float& v, float& w) {
  m = __fmaf_rn(b1, m, __fmul_rn(omb1, g));
  v = __fmaf_rn(b2, v, __fmul_rn(__fmul_rn(omb2, g), g));
  w = __fsub_rn(w, __fdiv_rn(__fmul_rn(lr, __fmul_rn(m, ibc1)), __fadd_rn(__fsqrt_rn(__fmul_rn(v, ibc2)), eps)));
}

// Where flat parameter p lives in the weight image: *bf16 = byte offset of its bf16 copy (or -1),
// *f32 / *f32b = float indices into the fp32 block (or -1).
__device__ __forceinline__ void img_pos(const PpoTcArgs& a, int p, int* bf16, int* f32, int* f32b) {
  *bf16 = -1;
  *f32 = -1;
  *f32b = -1;
  const int S = a.S, A = a.A;
  auto col_of = [&](int k) { return k < a.npriv ? k : 32 + (k - a.npriv); };
  for (int net = 0; net < 2; ++net) {
    const int* w = net ? a.c_w : a.a_w;
    const int o0 = net ? 64 : 0;
    int i = p - w[0];
    if (i >= 0 && i < (S + 1) * 64) {  // W1 [S][64], b1 [64]
      const int k = i / 64, o = i % 64;
      *bf16 = (int)core_off(o0 + o, k < S ? col_of(k) : a.ones_col, 128);
      return;
    }
    i = p - w[1];
    if (i >= 0 && i < 65 * 64) {  // W2 [64][64], b2 [64]
      const int k = i / 64, o = i % 64;
      if (k < 64)
        *bf16 = (int)(kImgW1 + (net ? 8192u : 0u) + core_off(k, o, 64));
      else
        *f32 = kFb2 + o0 + o;
      return;
    }
    const int nout = net ? 1 : A;
    i = p - w[2];
    if (i >= 0 && i < 65 * nout) {  // W3 [64][nout], b3 [nout]
      const int k = i / nout, o = i % nout;
      if (k < 64) {
        *bf16 = (int)(kImgW1 + (net ? 20480u : 16384u) + core_off(k, o, 64));
        if (net) *f32 = kFw3c + k;
      } else {
        *f32 = net ? kFb3c : kFb3a + o;
      }
      return;
    }
  }
  if (p >= a.log_std && p < a.log_std + A) *f32 = kFls + (p - a.log_std);
}

__device__ __forceinline__ void img_store(const PpoTcArgs& a, uint8_t* img, int p, float w) {
  int b, f, f2;
  img_pos(a, p, &b, &f, &f2);
  if (b >= 0) *reinterpret_cast<__nv_bfloat16*>(img + b) = __float2bfloat16_rn(w);
  float* fb = reinterpret_cast<float*>(img + kImgW1 + 22528);
  if (f >= 0) fb[f] = w;
  if (f2 >= 0) fb[f2] = w;
}

// 16 consecutive accumulator columns of this thread's TMEM lane
__device__ __forceinline__ void tmem16(uint32_t taddr, float* v) { tc::tmem_ld16(taddr, v); }

// a row's 64 columns [c0, c0+64) -> tanh(. + add[c]) -> bf16 into an R=128 core-form matrix at col cd
__device__ __forceinline__ void epi_tanh64(uint32_t tl, const float* add, uint8_t* dst, int row, int cd) {
#pragma unroll 1
  for (int c = 0; c < 64; c += 16) {
    float v[16];
    tmem16(tl + c, v);
    uint32_t pk[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      float z0 = v[2 * j], z1 = v[2 * j + 1];
      if (add) tc::add2(z0, z1, add[c + 2 * j], add[c + 2 * j + 1]);
      pk[j] = tc::pack_bf16(tc::tanh_fast(z0), tc::tanh_fast(z1));
    }
    *reinterpret_cast<uint4*>(dst + core_off(row, cd + c, 128)) = make_uint4(pk[0], pk[1], pk[2], pk[3]);
    *reinterpret_cast<uint4*>(dst + core_off(row, cd + c + 8, 128)) = make_uint4(pk[4], pk[5], pk[6], pk[7]);
  }
}

__device__ __forceinline__ float bf_lo(uint32_t w) { return __uint_as_float(w << 16); }
__device__ __forceinline__ float bf_hi(uint32_t w) { return __uint_as_float(w & 0xffff0000u); }

// delta = D[c] * (1 - h^2) with h the bf16 activations at `hsrc` (same row / columns)
__device__ __forceinline__ void epi_delta64(uint32_t tl, const uint8_t* hsrc, uint8_t* dst, int row, int cd) {
#pragma unroll 1
  for (int c = 0; c < 64; c += 16) {
    float v[16];
    tmem16(tl + c, v);
    const uint4 h0 = *reinterpret_cast<const uint4*>(hsrc + core_off(row, cd + c, 128));
    const uint4 h1 = *reinterpret_cast<const uint4*>(hsrc + core_off(row, cd + c + 8, 128));
    const uint32_t hw[8] = {h0.x, h0.y, h0.z, h0.w, h1.x, h1.y, h1.z, h1.w};
    uint32_t pk[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const float a0 = bf_lo(hw[j]), a1 = bf_hi(hw[j]);
      pk[j] = tc::pack_bf16(v[2 * j] * (1.f - a0 * a0), v[2 * j + 1] * (1.f - a1 * a1));
    }
    *reinterpret_cast<uint4*>(dst + core_off(row, cd + c, 128)) = make_uint4(pk[0], pk[1], pk[2], pk[3]);
    *reinterpret_cast<uint4*>(dst + core_off(row, cd + c + 8, 128)) = make_uint4(pk[4], pk[5], pk[6], pk[7]);
  }
}

struct Pipe {
  uint64_t* mbar;
  uint32_t phase;
  __device__ __forceinline__ void wait() {
    tc::mbar_wait(mbar, phase);
    phase ^= 1;
    tc::fence_after_sync();
  }
};

// generic smem writes -> async proxy, TMEM reads done, then the CTA barrier
__device__ __forceinline__ void publish() {
  tc::fence_proxy_async();
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
}

__global__ void __launch_bounds__(kThreads, 1) ppo_tc_kernel(const PpoTcArgs a) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ __align__(8) uint64_t s_mma, s_img;
  __shared__ uint32_t s_tmem;
  __shared__ uint32_t s_flags[8];  // gate parts of the cluster's CTAs (written over DSMEM)
  __shared__ float s_red[2][40];   // head-epilogue column sums (two row halves)
  __shared__ float s_db3[33];      // column sums of d3 (actor 0..31, critic 32)
  __shared__ double s_loss[3];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int C = a.C;
  const uint32_t rank = tc::cluster_ctarank();
  uint32_t chain_id;
  asm volatile("mov.u32 %0, %%clusterid.x;" : "=r"(chain_id));
  const PpoTcChain ch = a.chains[chain_id];
  const uint32_t sbase = tc::smem_u32(smem);
  uint8_t* img = ch.img;
  float* f32 = reinterpret_cast<float*>(smem + kOffF32);
  float* rows_f = reinterpret_cast<float*>(smem + kOffRows);  // [0] old_lp [1] adv [2] ret [3] dv
  uint32_t* ridx = reinterpret_cast<uint32_t*>(smem + kOffRidx);
  // TMEM lane (= row or output index) and column half of this thread
  const int lrow = 32 * (warp & 3) + lane, half = warp >> 2;

  if (warp == 0) tc::tmem_alloc(&s_tmem, 512);
  if (tid == 0) {
    tc::mbar_init(&s_mma, 1);
    tc::mbar_init(&s_img, 1);
  }
  if (tid < 8) s_flags[tid] = 0;
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t tbase = s_tmem;
  const uint32_t tl = tbase + ((uint32_t)(32 * (warp & 3)) << 16);  // this warp's lane quarter
  Pipe mma{&s_mma, 0}, imgp{&s_img, 0};

  // parameter slice of this CTA (reduction / Adam / image entries)
  const int chunk = ((a.P + C - 1) / C + 3) & ~3;
  const int p_lo = (int)rank * chunk, p_hi = min(a.P, p_lo + chunk);
  const float b1 = (float)a.b1, b2 = (float)a.b2, omb1 = (float)(1.0 - a.b1), omb2 = (float)(1.0 - a.b2);
  int64_t t = *ch.t;

  // ---- prologue: this slice's entries of the weight image from the master weights ----
  for (int p = p_lo + tid; p < p_hi; p += kThreads) img_store(a, img, p, ch.params[p]);
  asm volatile("fence.proxy.async.global;" ::: "memory");
  cluster_arrive();

  // gather (gather_minibatch ppo.hpp:83-103) of step st into X_hi / X_lo and the row scalars
  auto gather = [&](int64_t st) {
    const int q = tid & 127, hh = tid >> 7;
    const int qg = (int)rank * kRows + q;
    const bool valid = qg < a.mb;
    uint32_t i = 0;
    const float* prv = nullptr;
    const float* rest = nullptr;
    if (valid) {
      i = mb_index(a, ch, st, (uint32_t)qg);
      if (a.obs_mode == 1) {
        prv = a.obs + (size_t)i * a.Sp;
        rest = a.feat + (size_t)a.row[i / a.N] * a.F;
      } else {
        prv = a.obs + (size_t)i * a.S;
        rest = prv + a.npriv;
      }
    }
    if (hh == 0) {
      ridx[q] = valid ? i : 0xffffffffu;
      const double mean = a.advstat[0], denom = a.advstat[1];
      rows_f[q] = valid ? a.logp[i] : 0.f;
      rows_f[128 + q] = valid ? (float)(((double)a.adv[i] - mean) / denom) : 0.f;
      rows_f[256 + q] = valid ? a.ret[i] : 0.f;
    }
#pragma unroll 1
    for (int ck = hh * 12; ck < hh * 12 + 12; ++ck) {
      float x[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int c = ck * 8 + j;
        float v = 0.f;
        if (valid) {
          if (c < 32)
            v = (c < a.npriv) ? __ldg(prv + c) : 0.f;
          else if (c < 32 + a.nrest)
            v = __ldg(rest + (c - 32));
          else if (c == a.ones_col)
            v = 1.f;
        }
        x[j] = v;
      }
      uint32_t hi[4], lo[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        hi[j] = tc::pack_bf16(x[2 * j], x[2 * j + 1]);
        lo[j] = tc::pack_bf16(x[2 * j] - bf_lo(hi[j]), x[2 * j + 1] - bf_hi(hi[j]));
      }
      const uint32_t off = core_off(q, ck * 8, 128);
      *reinterpret_cast<uint4*>(smem + kOffXhi + off) = make_uint4(hi[0], hi[1], hi[2], hi[3]);
      *reinterpret_cast<uint4*>(smem + kOffRB + off) = make_uint4(lo[0], lo[1], lo[2], lo[3]);
    }
  };
  auto load_image = [&]() {
    if (tid == 0) {
      tc::fence_proxy_async();
      tc::mbar_arrive_expect_tx(&s_img, kImgW1 + kImgRest);
      constexpr uint32_t kChunk = 16384;
      for (uint32_t o = 0; o < kImgW1; o += kChunk)
        tc::bulk_g2s(smem + kOffRC + o, img + o, min(kChunk, kImgW1 - o), &s_img);
      for (uint32_t o = 0; o < kImgRest; o += kChunk)
        tc::bulk_g2s(smem + kOffRE + o, img + kImgW1 + o, min(kChunk, kImgRest - o), &s_img);
    }
  };

  gather(0);
  cluster_wait();  // the initial image is complete in global memory
  load_image();

  int fail_code = 0, fail_detail = 0;
  for (int64_t st = 0; st < a.steps; ++st) {
    imgp.wait();
    publish();  // X (gather) visible to the tensor core
    // ---- L1: D[0,128) = X_hi . W1 + X_lo . W1 ----
    if (tid == 0) {
      mma_chain(tbase + 0, sbase + kOffXhi, 128, 0, sbase + kOffRC, 128, 0, kXC / 16, 128, false);
      mma_chain(tbase + 0, sbase + kOffRB, 128, 0, sbase + kOffRC, 128, 0, kXC / 16, 128, true);
      tc::mma_commit(&s_mma);
    }
    mma.wait();
    // ---- H1 = tanh(D) -> RC (W1 is consumed); ones of nothing: b2 enters in the epilogue ----
    epi_tanh64(tl + half * 64, nullptr, smem + kOffRC, lrow, half * 64);
    publish();
    if (tid == 0) {  // L2 actor / critic (W2 read MN-major: K = its rows = inputs)
      mma_chain(tbase + 128, sbase + kOffRC, 128, 0, sbase + kOffW2a, 64, 1, 4, 64, false);
      mma_chain(tbase + 192, sbase + kOffRC + 16384, 128, 0, sbase + kOffW2c, 64, 1, 4, 64, false);
      tc::mma_commit(&s_mma);
    }
    mma.wait();
    epi_tanh64(tl + 128 + half * 64, f32 + kFb2 + half * 64, smem + kOffH2, lrow, half * 64);
    publish();
    if (tid == 0) {  // heads: actor N = 32, critic N = 16 (column 0 used)
      mma_chain(tbase + 256, sbase + kOffH2, 128, 0, sbase + kOffW3a, 64, 1, 4, 32, false);
      mma_chain(tbase + 288, sbase + kOffH2 + 16384, 128, 0, sbase + kOffW3c, 64, 1, 4, 16, false);
      tc::mma_commit(&s_mma);
    }
    mma.wait();
    // ---- head gradients (detail::ppo_loss_grads ppo.hpp:126-167), one row per thread ----
    {
      float* scr = reinterpret_cast<float*>(smem + kOffBuf2);  // [128][40] fp32: dlog_std terms, losses
      const int r = lrow;
      const bool valid = ridx[r] != 0xffffffffu;
      const float inv_n = 1.f / (float)a.mb;
      uint8_t* d3 = smem + kOffBuf1;
      if (half == 0) {  // actor: mean, log-prob, ratio, clipped surrogate
        float mu[32];
        tmem16(tl + 256, mu);
        tmem16(tl + 256 + 16, mu + 16);
        float pl = 0.f;
        float g[32];
        if (valid) {
          const float* act = a.act + (size_t)ridx[r] * a.A;
          float lp = 0.f;
          float z[32];
#pragma unroll
          for (int d = 0; d < 32; ++d) {
            z[d] = 0.f;
            if (d < a.A) {
              const float ls = f32[kFls + d];
              const float m = mu[d] + f32[kFb3a + d];
              z[d] = (__ldg(act + d) - m) * __expf(-ls);
              lp += -0.5f * kLogTwoPiF - ls - 0.5f * z[d] * z[d];
            }
          }
          const float ratio = __expf(lp - rows_f[r]);
          const float adv = rows_f[128 + r];
          const float s1 = ratio * adv;
          const float s2 = fminf(fmaxf(ratio, 1.f - a.clip), 1.f + a.clip) * adv;
          pl = -fminf(s1, s2) * inv_n;
          const float dl = (s1 <= s2) ? -adv * ratio * inv_n : 0.f;  // ties flow (ppo.hpp:146)
#pragma unroll
          for (int d = 0; d < 32; ++d) {
            const float isig = (d < a.A) ? __expf(-f32[kFls + d]) : 0.f;
            g[d] = dl * z[d] * isig;                        // dL/dmu
            scr[r * 40 + d] = (d < a.A) ? dl * (z[d] * z[d] - 1.f) : 0.f;  // dL/dlog_std terms
          }
        } else {
#pragma unroll
          for (int d = 0; d < 32; ++d) {
            g[d] = 0.f;
            scr[r * 40 + d] = 0.f;
          }
        }
        scr[r * 40 + 32] = pl;
#pragma unroll
        for (int c = 0; c < 32; c += 8) {
          uint32_t pk[4];
#pragma unroll
          for (int j = 0; j < 4; ++j) pk[j] = tc::pack_bf16(g[c + 2 * j], g[c + 2 * j + 1]);
          *reinterpret_cast<uint4*>(d3 + core_off(r, c, 128)) = make_uint4(pk[0], pk[1], pk[2], pk[3]);
        }
      } else {  // critic: value error, dV
        float vv[16];
        tmem16(tl + 288, vv);
        float vl = 0.f, dv = 0.f;
        if (valid) {
          const float err = vv[0] + f32[kFb3c] - rows_f[256 + r];
          vl = err * err * inv_n;
          dv = a.vf * 2.f * err * inv_n;
        }
        rows_f[384 + r] = dv;
        scr[r * 40 + 33] = vl;
        // d3 columns [32, 128): dV in column 32, zeros
#pragma unroll
        for (int c = 32; c < 128; c += 8) {
          const uint32_t w0 = (c == 32) ? tc::pack_bf16(dv, 0.f) : 0u;
          *reinterpret_cast<uint4*>(d3 + core_off(r, c, 128)) = make_uint4(w0, 0u, 0u, 0u);
        }
      }
    }
    publish();
    // ---- d2a = d3a . W3a^T (K-major W3a: N = its rows); dW3^T = d3^T . H2 (both MN-major) ----
    if (tid == 0) {
      mma_chain(tbase + 256, sbase + kOffBuf1, 128, 0, sbase + kOffW3a, 64, 0, 2, 64, false);
      mma_chain(tbase + 0, sbase + kOffBuf1, 128, 1, sbase + kOffH2, 128, 1, 8, 128, false);
      tc::mma_commit(&s_mma);
    }
    // column sums while the MMAs run: the head-epilogue terms (dlog_std over rows, losses) and
    // db3 = column sums of d3 (the bf16 operand rows, as dW3 sees them)
    {
      const float* scr = reinterpret_cast<const float*>(smem + kOffBuf2);
      if (tid < 68) {
        const int c = tid % 34, hh = tid / 34;
        float s = 0.f;
        for (int r = hh * 64; r < hh * 64 + 64; ++r) s += scr[r * 40 + c];
        s_red[hh][c] = s;
      } else if (tid >= 128 && tid < 128 + 33) {
        const int c = tid - 128;
        float s = 0.f;
        for (int r = 0; r < 128; ++r)
          s += __bfloat162float(*reinterpret_cast<const __nv_bfloat16*>(smem + kOffBuf1 + core_off(r, c, 128)));
        s_db3[c] = s;
      }
    }
    mma.wait();
    __syncthreads();  // s_red complete; the scratch in BUF2 is dead
    // ---- d2 = (.) o (1 - H2^2): actor from TMEM, critic as dV x w3c ----
    if (half == 0) {
      epi_delta64(tl + 256, smem + kOffH2, smem + kOffBuf2, lrow, 0);
    } else {
      const float dv = rows_f[384 + lrow];
#pragma unroll 1
      for (int c = 0; c < 64; c += 8) {
        const uint4 hq = *reinterpret_cast<const uint4*>(smem + kOffH2 + core_off(lrow, 64 + c, 128));
        const uint32_t hw[4] = {hq.x, hq.y, hq.z, hq.w};
        uint32_t pk[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const float a0 = bf_lo(hw[j]), a1 = bf_hi(hw[j]);
          pk[j] = tc::pack_bf16(dv * f32[kFw3c + c + 2 * j] * (1.f - a0 * a0),
                                dv * f32[kFw3c + c + 2 * j + 1] * (1.f - a1 * a1));
        }
        *reinterpret_cast<uint4*>(smem + kOffBuf2 + core_off(lrow, 64 + c, 128)) = make_uint4(pk[0], pk[1], pk[2], pk[3]);
      }
    }
    publish();
    // ---- d1 pre-activations = d2 . W2^T (K-major W2: N = its rows); dW2^T = d2^T . H1 ----
    if (tid == 0) {
      mma_chain(tbase + 320, sbase + kOffBuf2, 128, 0, sbase + kOffW2a, 64, 0, 4, 64, false);
      mma_chain(tbase + 384, sbase + kOffBuf2 + 16384, 128, 0, sbase + kOffW2c, 64, 0, 4, 64, false);
      mma_chain(tbase + 128, sbase + kOffBuf2, 128, 1, sbase + kOffRC, 128, 1, 8, 128, false);
      tc::mma_commit(&s_mma);
    }
    mma.wait();
    epi_delta64(tl + 320 + half * 64, smem + kOffRC, smem + kOffBuf1, lrow, half * 64);
    publish();
    if (tid == 0) {  // dW1^T = d1^T . X_hi
      mma_chain(tbase + 256, sbase + kOffBuf1, 128, 1, sbase + kOffXhi, 128, 1, 8, 192, false);
      tc::mma_commit(&s_mma);
    }
    // bias gradients of layers 2 and 3: column sums of d2 (BUF2) and d3 (in BUF1 until dW1's d1
    // overwrote it -- so d3's sums are taken from the per-row values below instead)
    mma.wait();
    // ---- partials: TMEM -> this CTA's slab row in the flat parameter order ----
    float* slab = ch.slab + (size_t)rank * a.Pp;
    {
      const int o = lrow;  // TMEM lane = output index (actor 0-63 | critic 64-127; d3: actor 0..A-1, critic 32)
      // dW3^T [0,128): columns = H2 inputs (actor 0-63, critic 64-127)
#pragma unroll 1
      for (int c0 = half * 64; c0 < half * 64 + 64; c0 += 16) {
        float v[16];
        tmem16(tl + c0, v);
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          const int k = c0 + j;
          if (k < 64 && o < a.A) slab[a.a_w[2] + k * a.A + o] = v[j];
          if (k >= 64 && o == 32) slab[a.c_w[2] + (k - 64)] = v[j];
        }
      }
      // dW2^T [128,256)
#pragma unroll 1
      for (int c0 = half * 64; c0 < half * 64 + 64; c0 += 16) {
        float v[16];
        tmem16(tl + 128 + c0, v);
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          const int k = c0 + j;
          if (k < 64 && o < 64) slab[a.a_w[1] + k * 64 + o] = v[j];
          if (k >= 64 && o >= 64) slab[a.c_w[1] + (k - 64) * 64 + (o - 64)] = v[j];
        }
      }
      // dW1^T [256,448): columns = X columns
      const int* w1 = (o < 64) ? a.a_w : a.c_w;
      const int oo = o & 63;
#pragma unroll 1
      for (int c0 = half * 96; c0 < half * 96 + 96; c0 += 16) {
        float v[16];
        tmem16(tl + 256 + c0, v);
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          const int c = c0 + j;
          int k = -1;
          if (c < a.npriv) k = c;
          else if (c >= 32 && c < 32 + a.nrest) k = a.npriv + (c - 32);
          else if (c == a.ones_col) k = a.S;  // the bias b1 follows W1 [S][64]
          if (k >= 0) slab[w1[0] + k * 64 + oo] = v[j];
        }
      }
    }
    // db2 = column sums of d2 (BUF2, bf16, as dW2 sees them); db3, dlog_std, losses from above
    if (tid < 128) {
      float sum = 0.f;
      for (int r = 0; r < 128; ++r)
        sum += __bfloat162float(*reinterpret_cast<const __nv_bfloat16*>(smem + kOffBuf2 + core_off(r, tid, 128)));
      const int* w2 = (tid < 64) ? a.a_w : a.c_w;
      slab[w2[1] + 64 * 64 + (tid & 63)] = sum;
    } else if (tid < 128 + 34) {
      const int c = tid - 128;
      const float sum = s_red[0][c] + s_red[1][c];
      if (c < a.A) {
        slab[a.log_std + c] = sum;
        slab[a.a_w[2] + 64 * a.A + c] = s_db3[c];
      }
      if (c == 32) {
        slab[a.P] = sum;  // policy loss terms
        slab[a.c_w[2] + 64] = s_db3[32];
      }
      if (c == 33) slab[a.P + 1] = sum;  // value loss terms
    }
    tc::fence_before_sync();
    cluster_arrive();  // release: this CTA's slab row
    cluster_wait();
    // ---- reduce this CTA's parameter slice over the C slab rows (rank order), gate, Adam ----
    int bad = 0;
    for (int p = p_lo + tid; p < p_hi; p += kThreads) {
      float g = 0.f;
      for (int c = 0; c < C; ++c) g += __ldcg(ch.slab + (size_t)c * a.Pp + p);
      if (p >= a.log_std && p < a.log_std + a.A) g -= a.ent;  // ppo.hpp:157
      bad |= !isfinite(g);
      ch.grads[p] = g;
    }
    bad = __syncthreads_or(bad);
    if (tid == 0) {  // this CTA's gradient verdict to every CTA of the cluster (DSMEM)
      for (int c = 0; c < C; ++c) st_cluster_u32(tc::mapa_shared(&s_flags[rank], (uint32_t)c), (uint32_t)bad);
      // losses (every CTA sums them in the same order) -- the reference checks these first
      double pl = 0.0, vl = 0.0, en = 0.0;
      for (int c = 0; c < C; ++c) {
        pl += (double)__ldcg(ch.slab + (size_t)c * a.Pp + a.P);
        vl += (double)__ldcg(ch.slab + (size_t)c * a.Pp + a.P + 1);
      }
      for (int d = 0; d < a.A; ++d) en += 0.5 * (1.8378770664093454836 + 1.0) + (double)f32[kFls + d];  // nn.hpp:273-277
      s_loss[0] = pl;
      s_loss[1] = vl;
      s_loss[2] = en;
    }
    cluster_arrive();
    cluster_wait();
    {
      const double pl = s_loss[0], vl = s_loss[1], en = s_loss[2];
      int code = 0, detail = 0;
      if (!isfinite(pl)) { code = PRB_ERR_NUMERIC; detail = 10; }
      else if (!isfinite(vl)) { code = PRB_ERR_NUMERIC; detail = 11; }
      else if (!isfinite(en)) { code = PRB_ERR_NUMERIC; detail = 12; }
      else {
        for (int c = 0; c < C; ++c)
          if (s_flags[c]) { code = PRB_ERR_NUMERIC; detail = 0; }
      }
      if (code) {  // nn.hpp:169-171: nothing is updated; the update ends at the last accepted step
        fail_code = code;
        fail_detail = detail;
        break;
      }
      if (rank == 0 && tid == 0) {
        ch.stats[0] += pl;
        ch.stats[1] += vl;
        ch.stats[2] += en;
        ch.stats[3] += 1.0;
      }
    }
    ++t;
    {
      const float ibc1 = (float)(1.0 / (1.0 - pow(a.b1, (double)t)));
      const float ibc2 = (float)(1.0 / (1.0 - pow(a.b2, (double)t)));
      for (int p = p_lo + tid; p < p_hi; p += kThreads) {
        float m = ch.m[p], v = ch.v[p], w = ch.params[p];
        adam_param(b1, b2, omb1, omb2, ch.lr, a.eps, ibc1, ibc2, ch.grads[p], m, v, w);
        ch.m[p] = m;
        ch.v[p] = v;
        ch.params[p] = w;
        img_store(a, img, p, w);
      }
    }
    asm volatile("fence.proxy.async.global;" ::: "memory");
    cluster_arrive();  // the slice's image entries
    if (st + 1 < a.steps) gather(st + 1);  // overlaps the barrier
    cluster_wait();
    if (st + 1 < a.steps) load_image();
  }
  if (rank == 0 && tid == 0) {
    *ch.t = t;
    if (fail_code) {
      ch.status[0] = fail_code;
      ch.status[1] = fail_detail;
    }
  }
  tc::fence_before_sync();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc(tbase, 512);
  (void)fail_code;
}

}  // namespace

size_t ppo_tc_smem_bytes() { return kSmemBytes; }

void launch_ppo_tc(const PpoTcArgs& a, int nchains, cudaStream_t s) {
  ensure_smem(ppo_tc_kernel, kSmemBytes);
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3((unsigned)(a.C * nchains));
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = kSmemBytes;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = (unsigned)a.C;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  PRB_CUDA(cudaLaunchKernelEx(&cfg, ppo_tc_kernel, a));
}

}  // namespace prb
