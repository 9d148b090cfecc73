// ppo_tc.cu -- ppo_update (ppo.hpp:249-296) on the 5th-gen tensor cores, a group of C
// co-resident CTAs per learner.
//
// A learner's update is a chain of minibatch steps (gather_minibatch ppo.hpp:83-103 ->
// detail::ppo_loss_grads :116-188 -> adam_step nn.hpp:164-182).  Here the C = ceil(mb / 128)
// CTAs of one learner run the whole chain (every epoch, every minibatch) in one launch, with
// barriers among those C CTAs only (ChainBar), so several learners (pod.hpp:436-461, SURVEY.md
// §7 step 6) run at once, C CTAs each.  Per step, CTA c of a learner owns minibatch rows
// [128c, 128c + 128):
//
//   gather    X = [private features hi | rest | 1] per row as bf16 hi + lo pairs  [128 x 192]
//   L1        D = X_hi . W1_hi + X_lo . W1_hi + X_hi . W1_lo   (actor | critic in N = 128 MMAs;
//             b1 via the ones column; W1 as bf16 hi + lo pairs too)
//   L2        H1 = tanh(D);  D = H1_a . W2a,  D = H1_c . W2c        (+ b2 in the epilogue)
//   heads     H2 = tanh(D);  D = H2_a . W3a (N = 32),  D = H2_c . W3c (N = 16)
//   head grads (per row, fp32: log-prob, ratio, clipped surrogate with the tie rule of
//             ppo.hpp:146, value error)           -> d3 = [dmu / sigma-scaled | dV]
//   backward  d2 = (d3 . W3^T) o (1 - H2^2)  (actor by MMA, critic as an outer product)
//             d1 = (d2 . W2^T) o (1 - H1^2)
//   weight gradients, batch as the contraction dimension (both operands MN-major):
//             dW3^T = d3^T . H2,  dW2^T = d2^T . H1,  dW1^T = d1^T . X_hi   (fp32 in TMEM)
//   partials  TMEM -> this CTA's slab row (flat parameter order) + log_std / loss terms
//   learner barrier; CTA c sums the C slab rows of its 1/C parameter slice in rank order,
//   evaluates its part of the finiteness gate (losses first, then gradients, the reference's
//   order), publishes its gate part; if every part passed, Adam on its slice (fp32 master
//   weights, adam_param's explicit roundings) and the slice's entries of the bf16 weight image;
//   learner barrier; every CTA bulk-copies the image (122 KB) for the next step.
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
constexpr int kScr = 41;
// TMEM columns holding the tanh derivatives 1 - h^2 (packed bf16 pairs, 32 per half) of layer 2
// (consumed by the d2 epilogue before the d1 accumulator [320,448) is issued) and of layer 1
constexpr uint32_t kTD2 = 384, kTD1 = 448;  // fp32 head-epilogue scratch row stride (odd: conflict-free both ways)

// shared-memory map (bytes from the 1024-aligned dynamic base)
constexpr uint32_t kOffXhi = 0;                        // X_hi   [128][192]            49152
constexpr uint32_t kOffRB = 49152;                     // X_lo [128][192] | BUF1 + BUF2
constexpr uint32_t kOffBuf1 = kOffRB;                  // d3 / d1 [128][128]          32768
constexpr uint32_t kOffBuf2 = kOffRB + 32768;          // d2 [128][128] (+ fp32 reduce scratch)
constexpr uint32_t kOffRC = kOffRB + 65536;            // W1 image [128 out][192] | H1 [128][128]
constexpr uint32_t kOffAct = kOffRC + 32768;           // actions [128][32] fp32 (after L1: W1 dead)
constexpr uint32_t kOffH2 = kOffRC + 49152;            // H2 [128][128]               32768
constexpr uint32_t kOffRE = kOffH2 + 32768;            // W2a, W2c [64][64], W3a [64][32], W3c [64][16]
constexpr uint32_t kOffW2a = kOffRE, kOffW2c = kOffRE + 8192, kOffW3a = kOffRE + 16384, kOffW3c = kOffRE + 20480;
constexpr uint32_t kOffF32 = kOffRE + 22528;           // fp32 block (image tail)        1040
constexpr uint32_t kOffRows = kOffF32 + 1040;          // per-row old_lp, adv, ret, dv [4][128] fp32
constexpr uint32_t kOffRidx = kOffRows + 2048;         // per-row buffer index [128] u32
constexpr uint32_t kSmemBytes = kOffRidx + 512;
constexpr uint32_t kStageBytes = kOffRE;  // X_hi .. H2, dead during the reduction: slice staging
constexpr uint32_t kOffGather = 98304;    // the next rows' fp32 staging [128][784 B] (after X_hi / X_lo;
                                          // its last 2 KB overlap W2a, reloaded with the image)
// image (global) = W1 block | RE | fp32 block, the smem bytes [kOffRC, +49152) ++ [kOffRE, +23568)
// image (global) = W1 hi | W1 lo (bf16 pairs: W1 multiplies inputs of magnitude ~1e2, so the
// first layer needs ~16-bit weights as well as inputs) | W2a W2c W3a W3c | fp32 block
constexpr uint32_t kImgW1 = 49152, kImgRestOff = 2 * kImgW1, kImgRest = 22528 + 1040;
static_assert(kImgRestOff + kImgRest == (uint32_t)kPpoTcImgBytes, "image size");
static_assert(kOffGather + 128 * 784 + 64 <= kOffF32, "gather staging must end before the fp32 block");
// where W1 lo lands in shared memory for the L1 MMAs: K-steps 0-3 in the dead upper 16 KB of RB,
// K-steps 4-11 in H2's region (both free until L1 is done)
constexpr uint32_t kOffW1loA = kOffRB + 49152, kOffW1loB = kOffRC + 49152;
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

__device__ __forceinline__ void cp_async8(void* smem_dst, const void* gsrc) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(tc::smem_u32(smem_dst)), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_async4(void* smem_dst, const void* gsrc) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(tc::smem_u32(smem_dst)), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

// Barrier of a learner's C CTAs (co-resident by the cooperative launch): a monotonic arrival
// counter in global memory, released by thread 0 after a CTA barrier (cumulative: the CTA's
// writes before it), acquired by thread 0's spin, then a CTA barrier.  A thread-block cluster
// would give a hardware barrier and DSMEM, but only 15 clusters of 8 fit on a B200 at once
// (its GPC layout), so 16 learners -- configs[3]'s 8 pods x 2 -- would run in two waves.
struct ChainBar {
  uint32_t* ctr;
  uint32_t target;
  int C;
  __device__ __forceinline__ void arrive() {
    __syncthreads();
    if (threadIdx.x == 0) asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(ctr) : "memory");
    target += (uint32_t)C;
  }
  __device__ __forceinline__ void wait() {
    if (threadIdx.x == 0) {
      uint32_t v;
      unsigned long long t0 = 0;
      int polls = 0;
      do {
        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(ctr) : "memory");
        if ((++polls & 1023) == 0) barrier_watchdog(t0);
      } while ((int32_t)(v - target) < 0);
    }
    __syncthreads();
  }
};

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

// adam_step (nn.hpp:164-182) for one fp32 parameter.  The reference runs it in fp64; this path
// (bf16 operands, fp32 master weights) is held to a tolerance, not to the SIMT path's bits, so the
// square root and the division are the hardware approximations (~2 ulp) rather than the IEEE
// sequences: 16 parameters per thread per step, on the step's critical path.
__device__ __forceinline__ void adam_param(float b1, float b2, float omb1, float omb2, float lr, float eps, float ibc1,
                                           float ibc2, float g, float& m, float& v, float& w) {
  m = __fmaf_rn(b1, m, __fmul_rn(omb1, g));
  v = __fmaf_rn(b2, v, __fmul_rn(__fmul_rn(omb2, g), g));
  float sq;
  asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(sq) : "f"(v * ibc2));
  w = w - __fdividef(lr * (m * ibc1), sq + eps);
}

// Where flat parameter p lives in the weight image: *bf16 = byte offset of its bf16 copy (or -1),
// *f32 / *f32b = float indices into the fp32 block (or -1).
__host__ __device__ inline void img_pos(const PpoTcArgs& a, int p, int* bf16, int* f32, int* f32b) {
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
        *bf16 = (int)(kImgRestOff + (net ? 8192u : 0u) + core_off(k, o, 64));
      else
        *f32 = kFb2 + o0 + o;
      return;
    }
    const int nout = net ? 1 : A;
    i = p - w[2];
    if (i >= 0 && i < 65 * nout) {  // W3 [64][nout], b3 [nout]
      const int k = i / nout, o = i % nout;
      if (k < 64) {
        *bf16 = (int)(kImgRestOff + (net ? 20480u : 16384u) + core_off(k, o, 64));
        if (net) *f32 = kFw3c + k;
      } else {
        *f32 = net ? kFb3c : kFb3a + o;
      }
      return;
    }
  }
  if (p >= a.log_std && p < a.log_std + A) *f32 = kFls + (p - a.log_std);
}

__device__ __forceinline__ void img_store_at(uint8_t* img, int2 e, float w) {
  if (e.x >= 0) {
    const __nv_bfloat16 hi = __float2bfloat16_rn(w);
    *reinterpret_cast<__nv_bfloat16*>(img + e.x) = hi;
    if (e.x < (int)kImgW1)  // a W1 entry: its low half too
      *reinterpret_cast<__nv_bfloat16*>(img + kImgW1 + e.x) = __float2bfloat16_rn(w - __bfloat162float(hi));
  }
  float* fb = reinterpret_cast<float*>(img + kImgRestOff + 22528);
  const int f = e.y & 0xffff, f2 = (e.y >> 16) & 0xffff;
  if (f != 0xffff) fb[f] = w;
  if (f2 != 0xffff) fb[f2] = w;
}

__device__ __forceinline__ void img_store(const PpoTcArgs& a, uint8_t* img, int p, float w) {
  img_store_at(img, a.imgpos[p], w);
}

// 16 consecutive accumulator columns of this thread's TMEM lane
__device__ __forceinline__ void tmem16(uint32_t taddr, float* v) { tc::tmem_ld16(taddr, v); }

__device__ __forceinline__ float bf_lo(uint32_t w) { return __uint_as_float(w << 16); }
__device__ __forceinline__ float bf_hi(uint32_t w) { return __uint_as_float(w & 0xffff0000u); }

// tanh(z) and its derivative 1 - tanh(z)^2 = 4t / (1 + t)^2 with t = exp(-2|z|): accurate to a few
// ulp in RELATIVE terms even for saturated units, where 1 - h^2 from tanh.approx (absolute error
// ~5e-4) or from a rounded h would be noise (the backward multiplies by it, nn.hpp:122-127)
__device__ __forceinline__ void tanh_d(float z, float& h, float& d) {
  const float t = __expf(-2.f * fabsf(z));
  float r;  // 1 / (1 + t), t in (0, 1]: the approximate reciprocal is within 1 ulp
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(1.f + t));
  h = copysignf((1.f - t) * r, z);
  d = 4.f * t * r * r;
}

// a row's 64 accumulator columns -> tanh(. + add[c]) -> bf16 into an R=128 core-form matrix at col cd
// ... and the tanh derivatives 1 - h^2 (from the fp32 h) as packed bf16 pairs to TMEM at t_deriv.
// Four 16-column chunks in a rolled loop: the kernel is large, and fully unrolled epilogues
// stalled on instruction fetch (ncu no_instruction at the tanh lines).
__device__ __forceinline__ void epi_tanh64(uint32_t tl, const float* add, uint8_t* dst, int row, int cd,
                                           uint32_t t_deriv) {
#pragma unroll 1
  for (int c = 0; c < 64; c += 16) {
    float v[16];
    tc::tmem_ld16(tl + c, v);
    uint32_t pk[8], dpk[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      float z0 = v[2 * j], z1 = v[2 * j + 1];
      if (add) tc::add2(z0, z1, add[c + 2 * j], add[c + 2 * j + 1]);
      float h0, h1, d0, d1;
      tanh_d(z0, h0, d0);
      tanh_d(z1, h1, d1);
      pk[j] = tc::pack_bf16(h0, h1);
      dpk[j] = tc::pack_bf16(d0, d1);
    }
    *reinterpret_cast<uint4*>(dst + core_off(row, cd + c, 128)) = make_uint4(pk[0], pk[1], pk[2], pk[3]);
    *reinterpret_cast<uint4*>(dst + core_off(row, cd + c + 8, 128)) = make_uint4(pk[4], pk[5], pk[6], pk[7]);
    tc::tmem_st8(t_deriv + (c >> 1), dpk);
  }
}

// delta = D[c] * (1 - h^2), the derivatives read back from TMEM at t_deriv (packed bf16 pairs)
__device__ __forceinline__ void epi_delta64(uint32_t tl, uint32_t t_deriv, uint8_t* dst, int row, int cd) {
#pragma unroll 1
  for (int c = 0; c < 64; c += 16) {
    float v[16];
    tc::tmem_ld16(tl + c, v);
    uint32_t dw[8];
    tc::tmem_ld8(t_deriv + (c >> 1), dw);
    uint32_t pk[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) pk[j] = tc::pack_bf16(v[2 * j] * bf_lo(dw[j]), v[2 * j + 1] * bf_hi(dw[j]));
    *reinterpret_cast<uint4*>(dst + core_off(row, cd + c, 128)) = make_uint4(pk[0], pk[1], pk[2], pk[3]);
    *reinterpret_cast<uint4*>(dst + core_off(row, cd + c + 8, 128)) = make_uint4(pk[4], pk[5], pk[6], pk[7]);
  }
}

// column swizzle of the staged action rows (even: 8-byte pairs stay adjacent and aligned)
__device__ __forceinline__ int act_swz(int r) { return (r & 15) << 1; }

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

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__global__ void __launch_bounds__(kThreads, 1) ppo_tc_kernel(const PpoTcArgs a) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ __align__(8) uint64_t s_mma, s_img;
  __shared__ uint32_t s_tmem;
  __shared__ float s_red[2][40];   // head-epilogue column sums (two row halves)
  __shared__ float s_db3[33];      // column sums of d3 (actor 0..31, critic 32)
  __shared__ float s_isig[32];     // 1 / sigma_d = exp(-log_std_d) of the step (0 past A)
  __shared__ double s_lossc[2][8]; // the C CTAs' policy / value loss terms
  __shared__ uint2 s_next[kRows];  // the next step's rows: (buffer index | ~0, shared-feature row)
  __shared__ double s_loss[3];
  __shared__ int s_colk[kXC];
  __shared__ __align__(8) uint64_t s_red_bar;
  __shared__ __align__(8) uint64_t s_gat;  // the gather's bulk row copies (128 arrivals per phase)
  __shared__ uint32_t s_gsh[kRows];         // per staged row: private base | rest base << 8 (floats)
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int C = a.C;
  const uint32_t rank = blockIdx.x % (uint32_t)C, chain_id = blockIdx.x / (uint32_t)C;
  const PpoTcChain ch = a.chains[chain_id];
  ChainBar cbar{ch.sync, 0u, C};
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
    tc::mbar_init(&s_red_bar, 1);
    tc::mbar_init(&s_gat, kRows);
  }
  if (tid < kXC) {  // X column -> W1 input row (the ones column -> the bias row S), -1 for padding
    int k = -1;
    if (tid < a.npriv) k = tid;
    else if (tid >= 32 && tid < 32 + a.nrest) k = a.npriv + (tid - 32);
    else if (tid == a.ones_col) k = a.S;
    s_colk[tid] = k;
  }
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
  cbar.arrive();

  // gather (gather_minibatch ppo.hpp:83-103) of step st, in two halves.  gather_issue: thread q
  // (< 128) copies row q's features with 1-D bulk copies (the TMA engine: one instruction per row
  // segment instead of one 4-byte cp.async per element) from the 16-byte-aligned address at or
  // below the row's start, so the row lands in its 784-byte staging slot at a shift of 0-3 floats
  // (kept in s_gsh; the allocations are padded for the overhang); the row scalars go by 4-byte
  // cp.async straight to rows_f.  gather_convert (after the mbarrier, cp.async and a CTA
  // barrier): one row half per thread, branch-free selects -> the bf16 hi / lo X tiles.
  // Slot: obs_mode 1 = the private obs row at [0, 36) floats, the shared-feature row from 36;
  // obs_mode 0 = the whole obs row (private | rest contiguous).
  constexpr int kSlot = 196;  // floats (784 B, 16-byte multiple; 196 = 4 mod 32)
  float* gst = reinterpret_cast<float*>(smem + kOffGather);
  uint32_t gat_phase = 0;
  // the minibatch rows of step st resolved ahead of time (Feistel / injected permutation and the
  // shared-feature row, whose dependent loads would otherwise serialise the gather): s_next[q]
  auto resolve_rows = [&](int64_t st) {
    if (tid < kRows) {
      const int qg = (int)rank * kRows + tid;
      uint2 e = make_uint2(0xffffffffu, 0u);
      if (qg < a.mb) {
        e.x = mb_index(a, ch, st, (uint32_t)qg);
        if (a.obs_mode == 1) e.y = (uint32_t)ch.row[e.x / a.N];
      }
      s_next[tid] = e;
    }
  };
  auto gather_issue = [&]() {  // the rows in s_next (resolve_rows + a barrier before)
    if (tid < kRows) {
      const int q = tid;
      const uint2 e = s_next[q];
      float* slot = gst + q * kSlot;
      if (e.x != 0xffffffffu) {
        const uint32_t i = e.x;
        const int nobs = a.obs_mode == 1 ? a.Sp : a.S;  // floats of the obs row
        const uintptr_t po = reinterpret_cast<uintptr_t>(ch.obs + (size_t)i * nobs);
        const uintptr_t po0 = po & ~(uintptr_t)15;
        const int sh1 = (int)(po - po0) >> 2;
        const uint32_t b1 = (uint32_t)((4 * (nobs + sh1) + 15) & ~15);
        int sh2 = 0;
        uint32_t b2 = 0;
        uintptr_t pf0 = 0;
        if (a.obs_mode == 1) {
          const uintptr_t pf = reinterpret_cast<uintptr_t>(ch.feat + (size_t)e.y * a.F);
          pf0 = pf & ~(uintptr_t)15;
          sh2 = (int)(pf - pf0) >> 2;
          b2 = (uint32_t)((4 * (a.F + sh2) + 15) & ~15);
        }
        tc::mbar_arrive_expect_tx(&s_gat, b1 + b2);
        tc::bulk_g2s(slot, reinterpret_cast<const void*>(po0), b1, &s_gat);
        if (b2) tc::bulk_g2s(slot + 36, reinterpret_cast<const void*>(pf0), b2, &s_gat);
        ridx[q] = i;
        s_gsh[q] = (uint32_t)sh1 | ((uint32_t)(a.obs_mode == 1 ? 4 + sh2 : sh1) << 8);
        cp_async4(rows_f + q, ch.logp + i);
        cp_async4(rows_f + 128 + q, ch.adv + i);
        cp_async4(rows_f + 256 + q, ch.ret + i);
      } else {
        tc::mbar_arrive(&s_gat);
        ridx[q] = 0xffffffffu;
        s_gsh[q] = 0;
      }
    }
  };
  auto gather_wait = [&]() {  // the bulk rows and the scalar copies of gather_issue, then a barrier
    tc::mbar_wait(&s_gat, gat_phase);
    gat_phase ^= 1;
    cp_async_wait_all();
    __syncthreads();
  };
  auto gather_convert = [&]() {
    const int q = tid & 127, hh = tid >> 7;
    const bool valid = ridx[q] != 0xffffffffu;
    const float* slot = gst + q * kSlot;
    const int pb = (int)(s_gsh[q] & 0xff), rb = (int)(s_gsh[q] >> 8);  // private / rest bases
    const int npriv = a.npriv, rend = 32 + a.nrest, onec = a.ones_col;
#pragma unroll
    for (int ck = 0; ck < 12; ++ck) {
      uint32_t hi[4], lo[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        float x2[2];
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          const int c = hh * 96 + ck * 8 + 2 * j + u;
          const bool priv = c < 32;
          const int idx = (priv ? pb : rb) + c;  // rest column c sits at rb + c (see gather_issue)
          const bool use = priv ? (c < npriv) : (c < rend);
          const float v = slot[idx];  // always a shared-memory address (overhang lands in RE)
          const float d = (c == onec) ? 1.f : 0.f;
          x2[u] = valid ? (use ? v : d) : 0.f;
        }
        hi[j] = tc::pack_bf16(x2[0], x2[1]);
        lo[j] = tc::pack_bf16(x2[0] - bf_lo(hi[j]), x2[1] - bf_hi(hi[j]));
      }
      const uint32_t off = core_off(q, hh * 96 + ck * 8, 128);
      *reinterpret_cast<uint4*>(smem + kOffXhi + off) = make_uint4(hi[0], hi[1], hi[2], hi[3]);
      *reinterpret_cast<uint4*>(smem + kOffRB + off) = make_uint4(lo[0], lo[1], lo[2], lo[3]);
    }
    if (hh == 0) {
      const double mean = ch.advstat[0], denom = ch.advstat[1];
      rows_f[q] = valid ? rows_f[q] : 0.f;
      rows_f[128 + q] = valid ? (float)(((double)rows_f[128 + q] - mean) / denom) : 0.f;
      rows_f[256 + q] = valid ? rows_f[256 + q] : 0.f;
    }
  };
  auto load_image = [&]() {
    if (tid == 0) {
      tc::fence_proxy_async();
      tc::mbar_arrive_expect_tx(&s_img, kImgRestOff + kImgRest);
      constexpr uint32_t kChunk = 16384;
      for (uint32_t o = 0; o < kImgW1; o += kChunk)
        tc::bulk_g2s(smem + kOffRC + o, img + o, min(kChunk, kImgW1 - o), &s_img);
      tc::bulk_g2s(smem + kOffW1loA, img + kImgW1, 16384, &s_img);  // W1 lo K-steps 0-3
      for (uint32_t o = 0; o < 32768; o += kChunk)                  // and 4-11
        tc::bulk_g2s(smem + kOffW1loB + o, img + kImgW1 + 16384 + o, kChunk, &s_img);
      for (uint32_t o = 0; o < kImgRest; o += kChunk)
        tc::bulk_g2s(smem + kOffRE + o, img + kImgRestOff + o, min(kChunk, kImgRest - o), &s_img);
    }
  };

  resolve_rows(0);
  __syncthreads();
  gather_issue();
  gather_wait();
  gather_convert();
  cbar.wait();  // the initial image is complete in global memory
  load_image();

  int fail_code = 0, fail_detail = 0;
  // debug phase trace (PpoTcArgs::trace, PRB_DEBUG_KNOBS builds): globaltimer marks of step 8
  unsigned long long* trp = (a.trace && rank == 0 && chain_id == 0 && tid == 0) ? a.trace : nullptr;
  int64_t cur_step = -1;
#define TCMARK(i)                                   \
  do {                                              \
    if (trp && cur_step == 8) trp[(i)] = gtimer(); \
  } while (0)
  uint32_t red_phase = 0;  // parity of s_red_bar (one completion per staged piece, across steps)
  for (int64_t st = 0; st < a.steps; ++st) {
    cur_step = st;
    TCMARK(0);
    imgp.wait();
    if (tid < 32) s_isig[tid] = tid < a.A ? __expf(-f32[kFls + tid]) : 0.f;
    publish();  // X (gather) visible to the tensor core
    TCMARK(1);
    // ---- L1: D[0,128) = [actor | critic] in N = 128 MMAs (the W1 image holds both nets' output
    // rows): X_hi . W1_hi + X_lo . W1_hi + X_hi . W1_lo (the lo . lo term is below fp32 rounding) ----
    if (tid == 0) {
      const uint32_t idesc = tc::idesc_bf16_t(128, 128, 0, 0);
      mma_chain(tbase + 0, sbase + kOffXhi, 128, 0, sbase + kOffRC, 128, 0, kXC / 16, 128, false);
      mma_chain(tbase + 0, sbase + kOffRB, 128, 0, sbase + kOffRC, 128, 0, kXC / 16, 128, true);
      for (int j = 0; j < kXC / 16; ++j) {
        const uint32_t bb = j < 4 ? sbase + kOffW1loA + j * 4096 : sbase + kOffW1loB + (j - 4) * 4096;
        tc::mma_bf16(tbase, desc_k(sbase + kOffXhi + j * 4096, 128), desc_k(bb, 128), idesc, 1u);
      }
      tc::mma_commit(&s_mma);
    }
    if (st + 1 < a.steps) resolve_rows(st + 1);  // read by gather_issue at the end of this step
    // ---- H1 = tanh(D) -> RC once both halves' MMAs are done reading W1 (b1 came with the ones
    // column; b2 enters in the next epilogue); the rows' actions start streaming into RC's spare
    // 16 KB (cp.async, consumed by the head epilogue) ----
    mma.wait();
    TCMARK(2);
    tc::fence_before_sync();
    __syncthreads();  // W1 (in RC) is no longer read by the tensor core: H1 may overwrite it
    {  // actions of this CTA's rows: [128][32] fp32, element d of row r at column
       // d ^ act_swz(r) (the row-per-thread reads of the head epilogue would otherwise all hit
       // one bank); 8-byte copies (A even: pairs stay adjacent) or 4-byte; two threads per row
      float* sact = reinterpret_cast<float*>(smem + kOffAct);
      const int r = tid >> 1, sw = act_swz(r);
      const uint32_t i = ridx[r];
      if (i != 0xffffffffu) {
        const float* src = ch.act + (size_t)i * a.A;
        if ((a.A & 1) == 0) {
          for (int k = 2 * (tid & 1); k < a.A; k += 4) cp_async8(sact + r * 32 + (k ^ sw), src + k);
        } else {
          for (int k = tid & 1; k < a.A; k += 2) cp_async4(sact + r * 32 + (k ^ sw), src + k);
        }
      }
    }
    epi_tanh64(tl + half * 64, nullptr, smem + kOffRC, lrow, half * 64, tl + kTD1 + half * 32);
    publish();
    TCMARK(3);
    if (tid == 0) {  // L2 actor / critic (W2 read MN-major: K = its rows = inputs)
      mma_chain(tbase + 128, sbase + kOffRC, 128, 0, sbase + kOffW2a, 64, 1, 4, 64, false);
      mma_chain(tbase + 192, sbase + kOffRC + 16384, 128, 0, sbase + kOffW2c, 64, 1, 4, 64, false);
      tc::mma_commit(&s_mma);
    }
    mma.wait();
    TCMARK(4);
    epi_tanh64(tl + 128 + half * 64, f32 + kFb2 + half * 64, smem + kOffH2, lrow, half * 64, tl + kTD2 + half * 32);
    cp_async_wait_all();  // the action copies (visible to every thread after the barrier)
    publish();
    TCMARK(5);
    if (tid == 0) {  // heads: actor N = 32, critic N = 16 (column 0 used)
      mma_chain(tbase + 256, sbase + kOffH2, 128, 0, sbase + kOffW3a, 64, 1, 4, 32, false);
      mma_chain(tbase + 288, sbase + kOffH2 + 16384, 128, 0, sbase + kOffW3c, 64, 1, 4, 16, false);
      tc::mma_commit(&s_mma);
    }
    mma.wait();
    TCMARK(6);
    // ---- head gradients (detail::ppo_loss_grads ppo.hpp:126-167), one row per thread ----
    {
      float* scr = reinterpret_cast<float*>(smem + kOffBuf2);  // [128][kScr] fp32: dlog_std terms, losses
      const int r = lrow;
      const bool valid = ridx[r] != 0xffffffffu;
      const float inv_n = 1.f / (float)a.mb;
      uint8_t* d3 = smem + kOffBuf1;
      if (half == 0) {  // actor: mean, log-prob, ratio, clipped surrogate (rolled 8-dim chunks;
                        // z is staged in this row's scratch, then replaced by the dlog_std terms)
        const float* sact = reinterpret_cast<const float*>(smem + kOffAct) + r * 32;
        const int asw = act_swz(r);
        float* zr = scr + r * kScr;
        float lp = 0.f;
#pragma unroll 1
        for (int c = 0; c < 32; c += 8) {
          uint32_t mw[8];
          tc::tmem_ld8(tl + 256 + c, mw);
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const int d = c + j;
            float z = 0.f;
            if (valid && d < a.A) {
              const float ls = f32[kFls + d];
              const float m = __uint_as_float(mw[j]) + f32[kFb3a + d];
              z = (sact[d ^ asw] - m) * s_isig[d];
              lp += -0.5f * kLogTwoPiF - ls - 0.5f * z * z;
            }
            zr[d] = z;
          }
        }
        float pl = 0.f, dl = 0.f;
        if (valid) {
          const float ratio = __expf(lp - rows_f[r]);
          const float adv = rows_f[128 + r];
          const float s1 = ratio * adv;
          // std::clamp / std::min as the reference evaluates them (a NaN ratio propagates into the
          // loss and trips the gate, ppo.hpp:139-142, :169)
          const float lo = 1.f - a.clip, hi = 1.f + a.clip;
          const float cl = (ratio < lo) ? lo : ((hi < ratio) ? hi : ratio);
          const float s2 = cl * adv;
          pl = -((s2 < s1) ? s2 : s1) * inv_n;
          dl = (s1 <= s2) ? -adv * ratio * inv_n : 0.f;  // ties flow (ppo.hpp:146)
        }
#pragma unroll 1
        for (int c = 0; c < 32; c += 8) {
          uint32_t pk[4];
#pragma unroll
          for (int j = 0; j < 8; j += 2) {
            float g2[2];
#pragma unroll
            for (int u = 0; u < 2; ++u) {
              const int d = c + j + u;
              const float z = zr[d];
              g2[u] = valid ? dl * z * s_isig[d] : 0.f;                      // dL/dmu
              zr[d] = (valid && d < a.A) ? dl * (z * z - 1.f) : 0.f;       // dL/dlog_std terms
            }
            pk[j >> 1] = tc::pack_bf16(g2[0], g2[1]);
          }
          *reinterpret_cast<uint4*>(d3 + core_off(r, c, 128)) = make_uint4(pk[0], pk[1], pk[2], pk[3]);
        }
        zr[32] = pl;
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
        scr[r * kScr + 33] = vl;
        // d3 columns [32, 128): dV in column 32, zeros
#pragma unroll
        for (int c = 32; c < 128; c += 8) {
          const uint32_t w0 = (c == 32) ? tc::pack_bf16(dv, 0.f) : 0u;
          *reinterpret_cast<uint4*>(d3 + core_off(r, c, 128)) = make_uint4(w0, 0u, 0u, 0u);
        }
      }
    }
    publish();
    TCMARK(7);
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
        for (int r = hh * 64; r < hh * 64 + 64; ++r) s += scr[r * kScr + c];
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
    TCMARK(8);
    __syncthreads();  // s_red complete; the scratch in BUF2 is dead
    // ---- d2 = (.) o (1 - H2^2): actor from TMEM, critic as dV x w3c ----
    if (half == 0) {
      epi_delta64(tl + 256, tl + kTD2, smem + kOffBuf2, lrow, 0);
    } else {
      const float dv = rows_f[384 + lrow];
      uint32_t dw[32];
      tc::tmem_ld32(tl + kTD2 + 32, dw);
#pragma unroll 1
      for (int c = 0; c < 64; c += 8) {
        uint32_t pk[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const uint32_t w = dw[(c >> 1) + j];
          pk[j] = tc::pack_bf16(dv * f32[kFw3c + c + 2 * j] * bf_lo(w), dv * f32[kFw3c + c + 2 * j + 1] * bf_hi(w));
        }
        *reinterpret_cast<uint4*>(smem + kOffBuf2 + core_off(lrow, 64 + c, 128)) = make_uint4(pk[0], pk[1], pk[2], pk[3]);
      }
    }
    publish();
    TCMARK(9);
    // ---- d1 pre-activations = d2 . W2^T (K-major W2: N = its rows); dW2^T = d2^T . H1 ----
    if (tid == 0) {
      mma_chain(tbase + 320, sbase + kOffBuf2, 128, 0, sbase + kOffW2a, 64, 0, 4, 64, false);
      mma_chain(tbase + 384, sbase + kOffBuf2 + 16384, 128, 0, sbase + kOffW2c, 64, 0, 4, 64, false);
      mma_chain(tbase + 128, sbase + kOffBuf2, 128, 1, sbase + kOffRC, 128, 1, 8, 128, false);
      tc::mma_commit(&s_mma);
    }
    mma.wait();
    TCMARK(10);
    epi_delta64(tl + 320 + half * 64, tl + kTD1 + half * 32, smem + kOffBuf1, lrow, half * 64);
    publish();
    TCMARK(11);
    if (tid == 0) {  // dW1^T = d1^T . X_hi
      mma_chain(tbase + 256, sbase + kOffBuf1, 128, 1, sbase + kOffXhi, 128, 1, 8, 192, false);
      tc::mma_commit(&s_mma);
    }
    // ---- partials: TMEM -> this CTA's slab row in global memory, in the flat parameter order,
    // straight from registers (a warp's 32 lanes = 32 consecutive outputs: coalesced 128-byte
    // stores; no shared-memory staging and no bulk store to wait for).  dW3^T and dW2^T are
    // complete: they leave while the dW1 MMA runs ----
    float* flat = ch.slab + (size_t)rank * a.Pp;
    const int o = lrow;  // TMEM lane = output index (actor 0-63 | critic 64-127; d3: actor 0..A-1, critic 32)
    const int oo = o & 63;
    {
      // dW3^T [0,128): columns = H2 inputs (actor 0-63 | critic 64-127); half h reads its net's
      // block (tcgen05.ld is warp-collective: every lane loads, the owners store)
      {
        const bool mine = half == 0 ? o < a.A : o == 32;
        float* dst = half == 0 ? flat + a.a_w[2] + o : flat + a.c_w[2];
        const int stride = half == 0 ? a.A : 1;
#pragma unroll 1
        for (int c = 0; c < 64; c += 16) {
          float v[16];
          tc::tmem_ld16(tl + half * 64 + c, v);
          if (mine) {
#pragma unroll
            for (int j = 0; j < 16; ++j) dst[(c + j) * stride] = v[j];
          }
        }
      }
      // dW2^T [128,256): the net's block is lanes of that net x its own input columns
      {
        const bool mine = (half == 0) == (o < 64);
        float* dst = (o < 64 ? flat + a.a_w[1] : flat + a.c_w[1]) + oo;
#pragma unroll 1
        for (int c = 0; c < 64; c += 16) {
          float v[16];
          tc::tmem_ld16(tl + 128 + half * 64 + c, v);
          if (mine) {
#pragma unroll
            for (int j = 0; j < 16; ++j) dst[(c + j) * 64] = v[j];
          }
        }
      }
    }
    // db2 = column sums of d2 (BUF2, bf16, as dW2 sees them) while dW1 runs
    float db2 = 0.f;
    if (tid < 128)
      for (int r = 0; r < 128; ++r)
        db2 += __bfloat162float(*reinterpret_cast<const __nv_bfloat16*>(smem + kOffBuf2 + core_off(r, tid, 128)));
    // bias gradients of layers 2 and 3: column sums of d2 (BUF2) and d3 (in BUF1 until dW1's d1
    // overwrote it -- so d3's sums are taken from the per-row values below instead)
    mma.wait();
    TCMARK(12);
    {
      // dW1^T [256,448): columns = X columns -> W1 rows (s_colk), the ones column -> b1
      {
        float* dst = (o < 64 ? flat + a.a_w[0] : flat + a.c_w[0]) + oo;
#pragma unroll 1
        for (int c0 = half * 96; c0 < half * 96 + 96; c0 += 48) {
          uint32_t r[64];
          tc::tmem_ld16_nw(tl + 256 + c0, r);
          tc::tmem_ld16_nw(tl + 256 + c0 + 16, r + 16);
          tc::tmem_ld16_nw(tl + 256 + c0 + 32, r + 32);
          tc::tmem_wait_ld64(r);
#pragma unroll
          for (int j = 0; j < 48; ++j) {
            const int k = s_colk[c0 + j];
            if (k >= 0) dst[k * 64] = __uint_as_float(r[j]);
          }
        }
      }
    }
    TCMARK(18);
    tc::fence_before_sync();
    if (tid < 128) {
      const int* w2 = (tid < 64) ? a.a_w : a.c_w;
      flat[w2[1] + 64 * 64 + (tid & 63)] = db2;
    } else if (tid < 128 + 34) {
      const int c = tid - 128;
      const float sum = s_red[0][c] + s_red[1][c];
      if (c < a.A) {
        flat[a.log_std + c] = sum;
        flat[a.a_w[2] + 64 * a.A + c] = s_db3[c];
      }
      if (c == 32) {
        flat[a.P] = sum;  // policy loss terms
        flat[a.c_w[2] + 64] = s_db3[32];
      }
      if (c == 33) flat[a.P + 1] = sum;  // value loss terms
    }
    TCMARK(19);
    // generic-proxy stores -> the peers' bulk (async-proxy) reads after the barrier
    asm volatile("fence.proxy.async.global;" ::: "memory");
    TCMARK(20);
    TCMARK(13);
    tc::fence_before_sync();
    cbar.arrive();  // release: this CTA's slab row
    cbar.wait();
    TCMARK(14);
    // ---- reduce this CTA's parameter slice over the C slab rows (rank order), Adam (speculative),
    // gate.  The slice's C partial rows and its m / v / master weights are staged into shared
    // memory by bulk copies (the MMA operand regions are dead by now): one L2 round trip.  Adam's
    // results stay in the staging area and the bf16 image is written at once; one learner barrier
    // then both publishes the image and exchanges the gate, and only an accepted step's results
    // are stored to the master weights / moments (nn.hpp:169-171: a rejected step changes nothing;
    // the image is rebuilt from the master weights when the next update starts) ----
    // staging: m, v, w [piece] first, then the C partial rows [piece] (the gather of the next step
    // streams into kOffGather.. once the partial rows are consumed)
    const int piece = min(chunk, ((int)(kStageBytes / 4) / (C + 3)) & ~3);
    float* stw = reinterpret_cast<float*>(smem);  // m, v, w [piece] each
    float* stg = stw + 3 * (size_t)piece;         // [C][piece] partials; row 0 := the reduced g
    int bad = 0;
    const int npieces = (p_hi > p_lo) ? (p_hi - p_lo + piece - 1) / piece : 0;
    auto stage = [&](int pc, bool slab_rows, bool state) {
      if (tid == 0) {
        const int q0 = p_lo + pc * piece, cnt = min(piece, p_hi - q0);
        const uint32_t bytes = (uint32_t)(((cnt + 3) & ~3) * 4);
        tc::fence_proxy_async();  // earlier generic accesses of the staging area
        asm volatile("fence.proxy.async.global;" ::: "memory");  // the peers' slab rows (acquired by the barrier)
        tc::mbar_arrive_expect_tx(&s_red_bar, bytes * ((slab_rows ? C : 0) + (state ? 3 : 0)));
        if (slab_rows)
          for (int c = 0; c < C; ++c)
            tc::bulk_g2s(stg + (size_t)c * piece, ch.slab + (size_t)c * a.Pp + q0, bytes, &s_red_bar);
        if (state) {
          tc::bulk_g2s(stw, ch.m + q0, bytes, &s_red_bar);
          tc::bulk_g2s(stw + piece, ch.v + q0, bytes, &s_red_bar);
          tc::bulk_g2s(stw + 2 * (size_t)piece, ch.params + q0, bytes, &s_red_bar);
        }
      }
      tc::mbar_wait(&s_red_bar, red_phase);
      red_phase ^= 1;
    };
    const float ibc1 = (float)(1.0 / (1.0 - pow(a.b1, (double)(t + 1))));
    const float ibc2 = (float)(1.0 / (1.0 - pow(a.b2, (double)(t + 1))));
    auto adam_piece = [&](int pc) {  // staging rows C..C+2 := the updated m, v, w; image entries
      const int q0 = p_lo + pc * piece, cnt = min(piece, p_hi - q0);
      constexpr int kB = 8;  // parameters per thread whose image positions are loaded together
      for (int j0 = 0; j0 < cnt; j0 += kB * kThreads) {
        int2 pos[kB];
#pragma unroll
        for (int b = 0; b < kB; ++b) {
          const int j = j0 + b * kThreads + tid;
          pos[b] = (j < cnt) ? __ldg(a.imgpos + q0 + j) : make_int2(-1, -1);
        }
#pragma unroll
        for (int b = 0; b < kB; ++b) {
          const int j = j0 + b * kThreads + tid;
          if (j >= cnt) continue;
          float* sm_ = stw + j;
          float* sv_ = stw + piece + j;
          float* sw_ = stw + 2 * (size_t)piece + j;
          float m = *sm_, v = *sv_, w = *sw_;
          adam_param(b1, b2, omb1, omb2, ch.lr, a.eps, ibc1, ibc2, stg[j], m, v, w);
          *sm_ = m;
          *sv_ = v;
          *sw_ = w;
          img_store_at(img, pos[b], w);
        }
      }
    };
    auto commit_piece = [&](int pc) {  // an accepted step: the staged results to the master copies
      const int q0 = p_lo + pc * piece, cnt = min(piece, p_hi - q0);
      for (int j = tid; j < cnt; j += kThreads) {
        ch.m[q0 + j] = stw[j];
        ch.v[q0 + j] = stw[piece + j];
        ch.params[q0 + j] = stw[2 * (size_t)piece + j];
      }
    };
    for (int pc = 0; pc < npieces; ++pc) {
      stage(pc, true, npieces == 1);
      TCMARK(21);
      const int q0 = p_lo + pc * piece, cnt = min(piece, p_hi - q0);
#pragma unroll 2
      for (int j = tid; j < cnt; j += kThreads) {
        float part[8];
#pragma unroll
        for (int c = 0; c < 8; ++c) part[c] = (c < C) ? stg[(size_t)c * piece + j] : 0.f;
        float g = 0.f;
#pragma unroll
        for (int c = 0; c < 8; ++c)
          if (c < C) g += part[c];  // rank order
        const int p = q0 + j;
        if (p >= a.log_std && p < a.log_std + a.A) g -= a.ent;  // ppo.hpp:157
        bad |= !isfinite(g);
        stg[j] = g;  // row 0 now holds the reduced gradient
        ch.grads[p] = g;
      }
      if (npieces > 1) {  // Adam + commit need the gate first: the pieces are revisited below
        __syncthreads();
      } else {
        __syncthreads();
        TCMARK(22);
        adam_piece(0);
      }
    }
    if (tid >= 64 && tid < 64 + 2 * C) {  // the C CTAs' loss terms, one load each
      const int c = (tid - 64) >> 1, which = (tid - 64) & 1;
      s_lossc[which][c] = (double)__ldcg(ch.slab + (size_t)c * a.Pp + a.P + which);
    }
    bad = __syncthreads_or(bad);
    TCMARK(15);
    if (tid == 0) {  // this CTA's gradient verdict, read by every CTA of the learner after the barrier
      *reinterpret_cast<volatile uint32_t*>(ch.sync + 8 + rank) = (uint32_t)bad;
      // losses (every CTA sums them in the same order) -- the reference checks these first
      double pl = 0.0, vl = 0.0, en = 0.0;
      for (int c = 0; c < C; ++c) {
        pl += s_lossc[0][c];
        vl += s_lossc[1][c];
      }
      for (int d = 0; d < a.A; ++d) en += 0.5 * (1.8378770664093454836 + 1.0) + (double)f32[kFls + d];  // nn.hpp:273-277
      s_loss[0] = pl;
      s_loss[1] = vl;
      s_loss[2] = en;
    }
    TCMARK(23);
    asm volatile("fence.proxy.async.global;" ::: "memory");  // the image entries, to the next bulk copies
    TCMARK(24);
    const bool more = st + 1 < a.steps;
    // the next rows' copies fly across the barrier when the staged m / v / w leave the gather
    // area free (one piece, i.e. >= 5 CTAs per learner at the stock pod's size)
    const bool early = npieces == 1 && 3 * piece * 4 <= (int)kOffGather;
    if (more && early) gather_issue();
    TCMARK(25);
    cbar.arrive();
    cbar.wait();
    TCMARK(16);
    {
      const double pl = s_loss[0], vl = s_loss[1], en = s_loss[2];
      int code = 0, detail = 0;
      if (!isfinite(pl)) { code = PRB_ERR_NUMERIC; detail = 10; }
      else if (!isfinite(vl)) { code = PRB_ERR_NUMERIC; detail = 11; }
      else if (!isfinite(en)) { code = PRB_ERR_NUMERIC; detail = 12; }
      else {
        for (int c = 0; c < C; ++c)
          if (__ldcg(ch.sync + 8 + c)) { code = PRB_ERR_NUMERIC; detail = 0; }
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
    if (npieces == 1) {
      commit_piece(0);
    } else {  // large slices (few CTAs): re-stage the gradient and state piece by piece
      for (int pc = 0; pc < npieces; ++pc) {
        const int q0 = p_lo + pc * piece, cnt = min(piece, p_hi - q0);
        stage(pc, false, true);
        for (int j = tid; j < cnt; j += kThreads) stg[j] = __ldcg(ch.grads + q0 + j);
        __syncthreads();
        adam_piece(pc);
        __syncthreads();
        commit_piece(pc);
        __syncthreads();
      }
      asm volatile("fence.proxy.async.global;" ::: "memory");
      cbar.arrive();  // these image entries were written after the gate
      cbar.wait();
    }
    __syncthreads();  // the staging area is free: the next X tiles and the image may land
    if (more) {
      if (!early) gather_issue();
      gather_wait();
      TCMARK(26);
      gather_convert();
      TCMARK(27);
      load_image();
    }
    TCMARK(17);
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

namespace {
__global__ void ppo_tc_pos_kernel(const PpoTcArgs a, int2* out) {
  for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < a.P; p += gridDim.x * blockDim.x) {
    int b, f, f2;
    img_pos(a, p, &b, &f, &f2);
    out[p] = make_int2(b, (f < 0 ? 0xffff : f) | ((f2 < 0 ? 0xffff : f2) << 16));
  }
}
}  // namespace

void ppo_tc_image_positions(const PpoTcArgs& a, int2* d_out, cudaStream_t s) {
  ppo_tc_pos_kernel<<<(a.P + 255) / 256, 256, 0, s>>>(a, d_out);
  PRB_CHECK_LAUNCH();
}

void launch_ppo_tc(const PpoTcArgs& a, int nchains, cudaStream_t s) {
  ensure_smem(ppo_tc_kernel, kSmemBytes);
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3((unsigned)(a.C * nchains));
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = kSmemBytes;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;  // every CTA of a learner co-resident (its barrier)
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  int dev = 0, sms = 0, occ = 0;
  PRB_CUDA(cudaGetDevice(&dev));
  PRB_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  PRB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, ppo_tc_kernel, kThreads, kSmemBytes));
  const int per_wave = std::max(1, sms * std::max(occ, 1) / a.C);  // learners resident at once
  for (int c0 = 0; c0 < nchains; c0 += per_wave) {  // more learners than fit: waves
    PpoTcArgs w = a;
    w.chains = a.chains + c0;
    const int n = std::min(per_wave, nchains - c0);
    cfg.gridDim = dim3((unsigned)(a.C * n));
    PRB_CUDA(cudaLaunchKernelEx(&cfg, ppo_tc_kernel, w));
  }
}

}  // namespace prb
