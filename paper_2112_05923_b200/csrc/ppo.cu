// ppo.cu -- PPO update on device (ppo_update ppo.hpp:249-296,
// detail::ppo_loss_grads ppo.hpp:116-188, mlp_backward_accumulate
// nn.hpp:105-132, adam_step nn.hpp:164-182).
//
// One minibatch step = four stream-ordered kernels, all parameters and the
// whole rollout staying in HBM/L2:
//   1. ppo_fwd_delta (row-parallel): each CTA gathers R rows of the minibatch
//      (permutation computed on the fly: a keyed Feistel bijection of the
//      buffer, or the injected reference permutation), rebuilds the
//      observation (compact stock rows + shared feature row), stages the whole
//      actor+critic weight set in shared memory (row stride out+1), runs the
//      forward with cached activations, forms the clipped-surrogate / value /
//      entropy head gradients (subgradient ties as ppo.hpp:146) and
//      back-propagates the deltas; it writes every layer's input rows and
//      delta rows (plus the per-row log_std terms and losses) to a [mb x ...]
//      slab (a few MB, L2-resident).
//   2. ppo_grad (output-parallel): dW_l = H_{l-1}^T . delta_l (and db_l =
//      colsum(delta_l) in the k0 = 0 tiles; the flat layout stores b_l right
//      after W_l) in 64x64 output tiles x row splits; 4x4 register blocking,
//      fixed-order sums into a [splits x P] partial slab.
//   3. ppo_sum: one thread per parameter sums the split partials in split
//      order (deterministic); the last CTA evaluates the step's gate: losses
//      first, then gradients (reference order), advancing t / the counter.
//   4. adam (agent.cu), skipped by the gate so a non-finite step leaves the
//      state untouched (nn.hpp:169-171).
// The minibatch counter lives on device, so a run of steps is one CUDA graph.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "mlp_simt.cuh"
#include "ppo_tc.h"
#include "policy_internal.h"
#include "prb_internal.h"
#include "rng.cuh"
#include "tc.cuh"

using namespace prb;

namespace {

constexpr float kLogTwoPiF = 1.8378770664093454836f;
constexpr int kPpoThreads = 256;
constexpr size_t kSmemBudget = 220 * 1024;
constexpr int kGatherUnroll = 8;  // observation columns per lane loaded before any store (S <= 256 in one pass)

struct PpoArgs {
  const float* params;
  MlpDesc actor, critic;
  int log_std_off, A, P, Pext;
  // buffer (time-major, index = h*N + e)
  int obs_mode, S, Sp, K;
  const float* obs;
  const int32_t* row;
  const float* feat;
  const float* act;
  const float* logp;
  const float* adv;
  const float* ret;
  const double* advstat;
  uint32_t N;
  // minibatch schedule
  const uint32_t* perm;  // injected [epochs][n] device indices (nullable)
  uint64_t seed;
  uint32_t n;         // buffer length
  uint32_t nmb;       // full minibatches per epoch
  int bits;           // Feistel domain bits (even)
  int mb;             // minibatch rows
  int R;              // rows per CTA
  int stage;          // 1: weights staged in shared memory (ld = out + 1)
  int r8;             // 1: the rows-of-8 path (fwd_delta_r8): staged [W;b], warp-split reductions
  const int64_t* step;  // device minibatch counter (epoch = step / nmb)
  double clip, ent, vf;
  int32_t* status;
  int ldw;  // max hidden width rounded to 4
  // per-row slab written by ppo_fwd_delta: layer inputs and deltas, row-major [mb][width]
  float* slab;
  int hin_off[2][kMaxLayers];  // H_{l-1} rows ([mb][dims[l]]); l = 0 is the observation (shared)
  int del_off[2][kMaxLayers];  // delta_l rows ([mb][dims[l+1]])
  int ls_off, loss_off;        // [mb][A] log_std terms, [mb][2] policy / value loss terms
  unsigned long long* trace;   // debug (PRB_PPO_TRACE): clock64 phase marks of CTA (0, net), else null
  // persistent rows-of-8 update: [W;b] of both nets in the staged shared-memory layout (actor
  // blocks, then the critic's at img_c), kept current by the Adam phase, so phase A stages a
  // net with a few bulk async copies instead of ~5K per-thread cp.async (null: cp.async path)
  float* wimg;
  int img_c;
  int nospec;  // 1: Adam stored after the gate barrier (PRB_PPO_NOSPEC, A/B), else speculatively before it
  // persistent update: [2][mb] (buffer index, shared-feature row) of a step's minibatch rows,
  // resolved one step ahead by the CTAs that have no row block in phase A (null: mb_row inline)
  uint2* rtab;
};

// Keyed balanced-Feistel bijection on [0, 2^bits), cycle-walked into [0, n).
__device__ __forceinline__ uint32_t feistel_perm(uint32_t x, uint32_t n, int bits, uint64_t key) {
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

__device__ __forceinline__ uint32_t mb_row(const PpoArgs& a, int64_t step, uint32_t q) {
  const uint32_t epoch = (uint32_t)(step / a.nmb);
  const uint32_t pos = (uint32_t)(step % a.nmb) * (uint32_t)a.mb + q;
  if (a.perm) return a.perm[(size_t)epoch * a.n + pos];
  return feistel_perm(pos, a.n, a.bits, derive_seed2(a.seed, 0x50504fULL /*"PPO"*/, epoch));
}

// floats of one net's staged weight set: every layer at row stride out+1
// rows-of-8 staged row stride: out+4 when out is a multiple of 4 keeps rows 16-byte aligned
// (16-byte async copies; the backward reads 4 consecutive weights of a row as one LDS.128, and
// the 8 rows of a quarter-warp phase then sit 16*(out/4+1) bytes apart: distinct 16-byte bank
// groups as long as out/4+1 is odd, i.e. out = 0 mod 8); otherwise out+1 (scalar reads).
// Layer blocks are rounded up to 4 floats so every block starts 16-byte aligned.
__host__ __device__ inline int r8_ld(int out) { return (out & 3) ? out + 1 : out + 4; }
__host__ __device__ inline int r8_block(int in, int out) { return ((in + 1) * r8_ld(out) + 3) & ~3; }

__host__ __device__ inline size_t staged_floats(const MlpDesc& d, int r8 = 0) {
  size_t n = 0;
  for (int l = 0; l < d.nl; ++l)
    n += r8 ? (size_t)r8_block(d.dims[l], d.dims[l + 1]) : (size_t)d.dims[l] * (d.dims[l + 1] + 1);
  return (n + 3) & ~size_t(3);
}

// position of flat parameter p (a weight or bias of net d) in the net's staged r8 image, or -1
__device__ __forceinline__ int r8_img_pos(const MlpDesc& d, int p) {
  int base = 0;
  for (int l = 0; l < d.nl; ++l) {
    const int in = d.dims[l], out = d.dims[l + 1];
    const int i = p - d.off[l];
    if (i >= 0 && i < (in + 1) * out) {
      const int k = i / out;
      return base + k * r8_ld(out) + (i - k * out);
    }
    base += r8_block(in, out);
  }
  return -1;
}

constexpr int kR8Scratch = 8 * 8 * 64;  // rows-of-8 path: [warp][row][col] partial sums

struct Smem {
  float* w;  // staged weights of this CTA's net (nullptr when not staged)
  float* x;
  float* h0;  // post-activation outputs of layer 0; layer l follows at R8 * round4(dims[i+1]) per layer i < l
  float* d0;
  float* d1;
  float* actn;
  float* misc;  // [R8][4]: old_lp, adv_norm, ret, -
  float* tmp;   // [R8][ldA]
  float* loss;  // [R8]
  float* scratch;  // r8: [8 warps][8 rows][64 cols]
  float* ls;       // r8: [ldA] log_std of the step (actor)
};

// shared-memory carve-up of one CTA working on net `net` (0 actor, 1 critic)
__host__ __device__ inline size_t carve(const PpoArgs& a, int net, float* base, Smem* s) {
  const MlpDesc& d = net ? a.critic : a.actor;
  const int R8 = (a.R + 7) & ~7;
  const int ldx = (a.S + 3) & ~3;
  const int ldA = (a.A + 3) & ~3;
  size_t o = 0;
  auto take = [&](size_t n) {
    float* p = base ? base + o : nullptr;
    o += (n + 3) & ~size_t(3);
    return p;
  };
  float* w = a.stage ? take(staged_floats(d, a.r8)) : nullptr;
  if (s) s->w = w;
  float* x = take((size_t)R8 * ldx);
  if (s) s->x = x;
  for (int l = 0; l < d.nl; ++l) {
    float* p = take((size_t)R8 * ((d.dims[l + 1] + 3) & ~3));
    if (s && l == 0) s->h0 = p;
  }
  const int ldd = a.ldw > ldA ? a.ldw : ldA;
  float* d0 = take((size_t)R8 * ldd);
  float* d1 = take((size_t)R8 * ldd);
  float* actn = take((size_t)R8 * ldA);
  float* misc = take((size_t)R8 * 4);
  float* tmp = take((size_t)R8 * ldA);
  float* loss = take((size_t)R8);
  float* scratch = a.r8 ? take((size_t)kR8Scratch) : nullptr;
  float* ls = a.r8 ? take((size_t)ldA) : nullptr;
  if (s) {
    s->scratch = scratch;
    s->ls = ls;
    s->d0 = d0;
    s->d1 = d1;
    s->actn = actn;
    s->misc = misc;
    s->tmp = tmp;
    s->loss = loss;
  }
  return o * sizeof(float);
}

inline size_t carve_max(const PpoArgs& a) { return std::max(carve(a, 0, nullptr, nullptr), carve(a, 1, nullptr, nullptr)); }

// Weight locations for one net: staged copy (stride out+1) or the HBM blob (stride out).
__device__ __forceinline__ LayerPtrs layer_ptrs(const PpoArgs& a, const MlpDesc& d, float* staged_base) {
  LayerPtrs lp;
  float* cur = staged_base;
  for (int l = 0; l < d.nl; ++l) {
    const float* Wg = a.params + d.off[l];
    lp.B[l] = Wg + (size_t)d.dims[l] * d.dims[l + 1];
    if (staged_base) {
      lp.W[l] = cur;
      lp.ldw[l] = d.dims[l + 1] + 1;
      cur += (size_t)d.dims[l] * (d.dims[l + 1] + 1);
    } else {
      lp.W[l] = Wg;
      lp.ldw[l] = d.dims[l + 1];
    }
  }
  return lp;
}

__device__ __forceinline__ void stage_weights(const PpoArgs& a, const MlpDesc& d, float* dst) {
  for (int l = 0; l < d.nl; ++l) {
    const int in = d.dims[l], out = d.dims[l + 1], ld = out + 1;
    const float* src = a.params + d.off[l];
    // row k of W -> dst[k*ld ...]: lanes walk a row (coalesced reads, conflict-free writes)
    const int OJ = out < 32 ? out : 32;
    const int KT = kPpoThreads / 32;
    const int lane = threadIdx.x & 31, kt = threadIdx.x >> 5;
    // LDGSTS: every element in flight at once, no register round trip (waited in stage_wait())
    if (lane < OJ)
      for (int k = kt; k < in; k += KT)
        for (int j = lane; j < out; j += OJ)
          asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(
                           (uint32_t)__cvta_generic_to_shared(dst + k * ld + j)),
                       "l"(src + (size_t)k * out + j)
                       : "memory");
    dst += (size_t)in * ld;
  }
}

__device__ __forceinline__ void stage_wait() {
  asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;" ::: "memory");
}

// rows [q0, q0+nrows) of a [mb][round4(w)] slab array <- smem tile s (row stride lds); the
// padding columns are never written (zero since allocation)
__device__ __forceinline__ void store_rows_g(float* __restrict__ g, int w, const float* s, int lds, int nrows, int q0) {
  const int n = nrows * w, gld = (w + 3) & ~3;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const int r = i / w, c = i - r * w;
    g[(size_t)(q0 + r) * gld + c] = s[r * lds + c];
  }
}

// d_prev[r][k] = (sum_j d[r][j] W[k][j]) * (1 - a[r][k]^2)   (matmul_nt, nn.hpp:125-130)
__device__ __forceinline__ void delta_prev_tile(const float* s_d, int ldd, int out, const float* W, int ldw, int in,
                                                const float* s_a, int lda, float* s_dp, int ldp, int nrows) {
  int KT = 32;
  while (KT < in && KT < (int)blockDim.x) KT <<= 1;
  const int NRG = blockDim.x / KT;
  const int kk = threadIdx.x % KT, rg = threadIdx.x / KT;
  for (int r = rg; r < nrows; r += NRG) {
    const float* dr = s_d + r * ldd;
    for (int k = kk; k < in; k += KT) {
      const float* wr = W + (size_t)k * ldw;
      float acc = 0.0f;
      for (int j = 0; j < out; ++j) acc = fmaf(dr[j], wr[j], acc);
      const float av = s_a[r * lda + k];
      s_dp[r * ldp + k] = acc * (1.0f - av * av);
    }
  }
}

// blockIdx.y = net: the actor and the critic are independent through the forward,
// their heads and the backward, so each CTA carries one net (half the weights to stage).
// STAGED: the net's weights are copied to shared memory (every W access is an LDS);
// otherwise (nets too wide for the tile) they are read from L2.

// ============================================================================================
// Rows-of-8 path (R <= 8, every layer width <= 64, A <= 32; the stock 64x64 nets).  The
// per-kernel tile functions above keep one or two rows per thread, so every staged weight is
// re-read from shared memory for each row pair and the k-chains are as long as the layer input;
// here each warp owns a slice of the reduction dimension for ALL 8 rows and up to 64 columns
// (8 x 2 register accumulators, x read as float4 broadcasts), and the 8 warp partials are
// summed in fixed warp order (deterministic).  [W; b] are staged together ((in+1) rows at
// stride out+1, conflict-free for both the row walk of the forward and the column walk of
// the backward) with 16-byte global loads.
// ============================================================================================

// [W_l; b_l] of every layer -> dst rows of stride r8_ld(out) (bias = row `in`), asynchronously:
// 16-byte cp.async when the rows allow it, 4-byte otherwise; waited with stage_wait()
__device__ __forceinline__ void stage_weights_r8(const PpoArgs& a, const MlpDesc& d, float* dst) {
  // Each thread owns one column chunk and strides over rows, so the address arithmetic is one
  // division per layer instead of one per copy (the per-copy division made issuing the ~4.6K
  // copies of a 3-layer 64-wide actor take ~3 us, profiles/ppo_trace.py).
  const int tid = threadIdx.x, nt = blockDim.x;
  for (int l = 0; l < d.nl; ++l) {
    const int in = d.dims[l], out = d.dims[l + 1], ld = r8_ld(out);
    const float* src = a.params + d.off[l];
    if ((out & 3) == 0 && (reinterpret_cast<uintptr_t>(src) & 15) == 0 && (out >> 2) <= nt) {
      const int c4 = out >> 2, rows = nt / c4;  // rows per pass
      const int k0 = tid / c4, j = (tid - k0 * c4) << 2;
      if (k0 < rows)
        for (int k = k0; k <= in; k += rows)
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(
                           (uint32_t)__cvta_generic_to_shared(dst + k * ld + j)),
                       "l"(src + (size_t)k * out + j)
                       : "memory");
    } else if (out <= nt) {
      const int rows = nt / out;
      const int k0 = tid / out, j = tid - k0 * out;
      if (k0 < rows)
        for (int k = k0; k <= in; k += rows)
          asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(
                           (uint32_t)__cvta_generic_to_shared(dst + k * ld + j)),
                       "l"(src + (size_t)k * out + j)
                       : "memory");
    } else {
      const int n = (in + 1) * out;
      for (int i = tid; i < n; i += nt) {
        const int k = i / out, jj = i - k * out;
        asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(
                         (uint32_t)__cvta_generic_to_shared(dst + k * ld + jj)),
                     "l"(src + i)
                     : "memory");
      }
    }
    dst += r8_block(in, out);
  }
}

// scratch[w][r][c] = sum over this warp's slice of i of in[r][i] * Wt(i, c), r < 8, c < ncols <= 64,
// Wt(i, c) = W[i * ldw + c] (forward, TRANS = false) or W[c * ldw + i] (backward, TRANS = true).
// Warp w takes the groups of 4 i in [w*ng/8, (w+1)*ng/8); warp 7 also the nred % 4 tail.
template <bool TRANS>
__device__ __forceinline__ void r8_partials(const float* W, int ldw, const float* s_in, int ldi, int nred, int ncols,
                                            float* scratch) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int c0 = lane, c1 = lane + 32;
  const bool on0 = c0 < ncols, on1 = c1 < ncols;
  float acc0[8], acc1[8];
#pragma unroll
  for (int r = 0; r < 8; ++r) acc0[r] = acc1[r] = 0.0f;
  const int ng = nred >> 2;
  const int g0 = (w * ng) >> 3, g1 = ((w + 1) * ng) >> 3;
  for (int g = g0; g < g1; ++g) {
    const int i = 4 * g;
    float w0[4], w1[4];
    if (TRANS && (ldw & 3) == 0) {  // 16-byte row segments: one LDS.128 per column
      const float4 z4 = make_float4(0.f, 0.f, 0.f, 0.f);
      const float4 a4 = on0 ? *reinterpret_cast<const float4*>(W + c0 * ldw + i) : z4;
      const float4 b4 = on1 ? *reinterpret_cast<const float4*>(W + c1 * ldw + i) : z4;
      w0[0] = a4.x, w0[1] = a4.y, w0[2] = a4.z, w0[3] = a4.w;
      w1[0] = b4.x, w1[1] = b4.y, w1[2] = b4.z, w1[3] = b4.w;
    } else {
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        w0[u] = on0 ? (TRANS ? W[c0 * ldw + i + u] : W[(i + u) * ldw + c0]) : 0.0f;
        w1[u] = on1 ? (TRANS ? W[c1 * ldw + i + u] : W[(i + u) * ldw + c1]) : 0.0f;
      }
    }
#pragma unroll
    for (int r = 0; r < 8; ++r) {
      const float4 x = *reinterpret_cast<const float4*>(s_in + r * ldi + i);
      tc::fma2(acc0[r], acc1[r], x.x, w0[0], w1[0]);  // packed: the same per-column fmaf chain
      tc::fma2(acc0[r], acc1[r], x.y, w0[1], w1[1]);
      tc::fma2(acc0[r], acc1[r], x.z, w0[2], w1[2]);
      tc::fma2(acc0[r], acc1[r], x.w, w0[3], w1[3]);
    }
  }
  if (w == 7)
    for (int i = 4 * ng; i < nred; ++i) {
      const float wa = on0 ? (TRANS ? W[c0 * ldw + i] : W[i * ldw + c0]) : 0.0f;
      const float wb = on1 ? (TRANS ? W[c1 * ldw + i] : W[i * ldw + c1]) : 0.0f;
#pragma unroll
      for (int r = 0; r < 8; ++r) {
        tc::fma2(acc0[r], acc1[r], s_in[r * ldi + i], wa, wb);
      }
    }
  float* sc = scratch + w * 512;
#pragma unroll
  for (int r = 0; r < 8; ++r) {
    sc[r * 64 + c0] = acc0[r];
    sc[r * 64 + c1] = acc1[r];
  }
}

// sum of the 8 warp partials of output (r, c), in warp order
__device__ __forceinline__ float r8_sum(const float* scratch, int r, int c) {
  float v = 0.0f;
#pragma unroll
  for (int w = 0; w < 8; ++w) v += scratch[w * 512 + r * 64 + c];
  return v;
}

// rows [q0, q0+nrows) of a [mb][round4(w)] slab array <- smem rows (warp per row, no division)
__device__ __forceinline__ void store_rows_r8(float* __restrict__ g, int w, const float* s, int lds, int nrows, int q0) {
  const int lane = threadIdx.x & 31, gld = (w + 3) & ~3;
  for (int r = threadIdx.x >> 5; r < nrows; r += blockDim.x >> 5) {
    float* dst = g + (size_t)(q0 + r) * gld;
    const float* src = s + r * lds;
    for (int c = lane; c < w; c += 32) dst[c] = src[c];
  }
}

__device__ __forceinline__ void fwd_delta_r8(const PpoArgs& a, int bx, int net, int64_t step, float* smem,
                                             uint64_t* mbar = nullptr, uint32_t* mphase = nullptr,
                                             const uint2* rows = nullptr) {
  const MlpDesc& d = net ? a.critic : a.actor;
  unsigned long long* tr = (a.trace && bx == 0 && threadIdx.x == 0) ? a.trace + 16 * net : nullptr;
  int ntr = 0;
  auto mark = [&]() {
    if (tr && ntr < 16) tr[ntr++] = clock64();
  };
  mark();
  Smem s;
  carve(a, net, smem, &s);
  const int ldx = (a.S + 3) & ~3;
  const int A = a.A, ldA = (A + 3) & ~3;
  const int q0 = bx * 8;
  const int nrows = min(8, a.mb - q0);
  const double mean = a.advstat[0], denom = a.advstat[1];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  auto h_of = [&](int l) -> float* {
    float* p = s.h0;
    for (int i = 0; i < l; ++i) p += 8 * ((d.dims[i + 1] + 3) & ~3);
    return p;
  };
  auto ldh_of = [&](int l) { return (d.dims[l + 1] + 3) & ~3; };
  auto w_of = [&](int l) -> const float* {
    float* p = s.w;
    for (int i = 0; i < l; ++i) p += r8_block(d.dims[i], d.dims[i + 1]);
    return p;
  };
  if (mbar) {  // bulk async copies of the net's image (persistent update): 8 KB per lane of warp 0,
    // issued before the gather (the proxy fence would otherwise wait for the gather's loads)
    if (warp == 0) {
      const uint32_t bytes = (uint32_t)(staged_floats(d, 1) * sizeof(float));
      const char* src = reinterpret_cast<const char*>(a.wimg + (net ? a.img_c : 0));
      char* dst = reinterpret_cast<char*>(s.w);
      if (lane == 0) {
        tc::fence_proxy_async();  // this CTA's earlier generic reads of s.w before the async writes
        asm volatile("fence.proxy.async.global;" ::: "memory");  // image stores of the last Adam phase
        tc::mbar_arrive_expect_tx(mbar, bytes);
      }
      __syncwarp();
      constexpr uint32_t kChunk = 8192;
      for (uint32_t o = (uint32_t)lane * kChunk; o < bytes; o += 32 * kChunk)
        tc::bulk_g2s(dst + o, src + o, min(kChunk, bytes - o), mbar);
    }
  }
  mark();
  // ---- gather (gather_minibatch ppo.hpp:83-103): warp r gathers row r; its loads are issued
  // first, then the weight copies (asynchronous), then the gathered values are stored ----
  float xv[kGatherUnroll];
  float act = 0.f, lp0 = 0.f, advv = 0.f, retv = 0.f;
  const int r = warp;
  if (r < nrows) {
    uint32_t i;
    const float* fr = nullptr;
    if (rows) {  // resolved during the previous step
      const uint2 e = rows[q0 + r];
      i = e.x;
      if (a.obs_mode == 1) fr = a.feat + (size_t)e.y * (a.S - a.Sp);
    } else {
      i = mb_row(a, step, (uint32_t)(q0 + r));
      if (a.obs_mode == 1) fr = a.feat + (size_t)a.row[i / a.N] * (a.S - a.Sp);
    }
#pragma unroll
    for (int u = 0; u < kGatherUnroll; ++u) {
      const int c = lane + 32 * u;
      float v = 0.0f;
      if (c < a.S) {
        if (a.obs_mode == 1)
          v = (c < a.Sp) ? a.obs[(size_t)i * a.Sp + c] : fr[c - a.Sp];
        else
          v = a.obs[(size_t)i * a.S + c];
      }
      xv[u] = v;
    }
    for (int c = lane + 32 * kGatherUnroll; c < a.S; c += 32)  // wide observations
      s.x[r * ldx + c] = (a.obs_mode == 1) ? ((c < a.Sp) ? a.obs[(size_t)i * a.Sp + c] : fr[c - a.Sp])
                                           : a.obs[(size_t)i * a.S + c];
    if (net == 0) {
      act = (lane < A) ? a.act[(size_t)i * A + lane] : 0.0f;
      if (lane == 0) {
        lp0 = a.logp[i];
        advv = a.adv[i];
      }
    } else if (lane == 0) {
      retv = a.ret[i];
    }
  }
  if (!mbar) stage_weights_r8(a, d, s.w);
  mark();
  if (net == 0)
    for (int dd = threadIdx.x; dd < A; dd += blockDim.x) s.ls[dd] = a.params[a.log_std_off + dd];
  if (r < nrows) {
#pragma unroll
    for (int u = 0; u < kGatherUnroll; ++u)
      if (lane + 32 * u < a.S) s.x[r * ldx + lane + 32 * u] = xv[u];
    if (net == 0 && lane < A) s.actn[r * ldA + lane] = act;
    if (lane == 0) {
      s.misc[r * 4 + 0] = lp0;
      s.misc[r * 4 + 1] = (float)(((double)advv - mean) / denom);
      s.misc[r * 4 + 2] = retv;
    }
  }
  mark();
  if (mbar) {
    tc::mbar_wait(mbar, *mphase);
    *mphase ^= 1u;
  } else {
    stage_wait();
  }
  mark();
  __syncthreads();
  mark();
  // ---- forward with caches (mlp_forward nn.hpp:63-85) ----
  {
    const float* in = s.x;
    int ldi = ldx;
#pragma unroll 1
    for (int l = 0; l < d.nl; ++l) {
      const int din = d.dims[l], out = d.dims[l + 1];
      const float* W = w_of(l);
      r8_partials<false>(W, r8_ld(out), in, ldi, din, out, s.scratch);
      __syncthreads();
      float* o = h_of(l);
      const int ldo = ldh_of(l);
      const float* b = W + din * r8_ld(out);
      for (int e = threadIdx.x; e < 8 * out; e += blockDim.x) {
        const int rr = e / out, c = e - rr * out;
        const float z = r8_sum(s.scratch, rr, c) + b[c];
        o[rr * ldo + c] = (l + 1 < d.nl) ? tanhf(z) : z;
      }
      __syncthreads();
      in = o;
      ldi = ldo;
      mark();
    }
  }
  // layer inputs for the gradient GEMMs: the observation (actor CTAs) and every hidden activation
  if (net == 0) store_rows_r8(a.slab + a.hin_off[0][0], a.S, s.x, ldx, nrows, q0);
  for (int l = 1; l < d.nl; ++l) store_rows_r8(a.slab + a.hin_off[net][l], d.dims[l], h_of(l - 1), ldh_of(l - 1), nrows, q0);
  mark();
  // ---- per-row losses and head gradients (ppo.hpp:128-167): warp r = row r ----
  const float inv_n = 1.0f / (float)a.mb;
  float* head = h_of(d.nl - 1);
  const int ldm = ldh_of(d.nl - 1);
  if (net == 0) {
    if (r < nrows) {
      const bool on = lane < A;
      const float ls = on ? s.ls[lane] : 0.0f;
      const float isig = expf(-ls);
      const float z = on ? (s.actn[r * ldA + lane] - head[r * ldm + lane]) * isig : 0.0f;  // (a - mu) / sigma
      float lpv = on ? (-0.5f * kLogTwoPiF - ls) - 0.5f * z * z : 0.0f;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) lpv += __shfl_xor_sync(0xffffffffu, lpv, o);
      const float ratio = expf(lpv - s.misc[r * 4 + 0]);
      const float adv = s.misc[r * 4 + 1];
      const float surr1 = ratio * adv;
      const float lo = (float)(1.0 - a.clip), hi = (float)(1.0 + a.clip);
      const float clipped = (ratio < lo) ? lo : ((hi < ratio) ? hi : ratio);  // std::clamp
      const float surr2 = clipped * adv;
      const float dl_dlp = (surr1 <= surr2) ? -adv * ratio * inv_n : 0.0f;  // ppo.hpp:146
      if (on) {
        head[r * ldm + lane] = dl_dlp * (z * isig);  // dmean = dL/dlp * z / sigma, in place
        s.tmp[r * ldA + lane] = dl_dlp * (z * z - 1.0f);
      }
      if (lane == 0) s.loss[r] = -((surr2 < surr1) ? surr2 : surr1) * inv_n;  // std::min (NaN-propagating)
    }
  } else {
    for (int rr = threadIdx.x; rr < nrows; rr += blockDim.x) {
      const float err = head[rr * ldm] - s.misc[rr * 4 + 2];
      s.loss[rr] = err * err * inv_n;
      head[rr * ldm] = (float)a.vf * 2.0f * err * inv_n;  // dV, in place
    }
  }
  __syncthreads();
  mark();
  store_rows_r8(a.slab + a.del_off[net][d.nl - 1], d.dims[d.nl], head, ldm, nrows, q0);
  if (net == 0) store_rows_r8(a.slab + a.ls_off, A, s.tmp, ldA, nrows, q0);
  for (int rr = threadIdx.x; rr < nrows; rr += blockDim.x) a.slab[a.loss_off + (size_t)(q0 + rr) * 2 + net] = s.loss[rr];
  mark();
  // ---- backward deltas (mlp_backward_accumulate nn.hpp:105-132, the matmul_nt half) ----
  const int ldp = a.ldw > ldA ? a.ldw : ldA;
  const float* delta = head;
  int ldd = ldm;
  for (int l = d.nl - 1; l >= 1; --l) {
    const int in = d.dims[l], out = d.dims[l + 1];
    float* dp = (delta == s.d0) ? s.d1 : s.d0;
    r8_partials<true>(w_of(l), r8_ld(out), delta, ldd, out, in, s.scratch);
    __syncthreads();
    const float* act_in = h_of(l - 1);
    const int lda = ldh_of(l - 1);
    for (int e = threadIdx.x; e < 8 * in; e += blockDim.x) {
      const int rr = e / in, k = e - rr * in;
      const float av = act_in[rr * lda + k];
      dp[rr * ldp + k] = r8_sum(s.scratch, rr, k) * (1.0f - av * av);
    }
    __syncthreads();
    mark();
    store_rows_r8(a.slab + a.del_off[net][l - 1], in, dp, ldp, nrows, q0);
    delta = dp;
    ldd = ldp;
    mark();
  }
}

// (bx, net) is the virtual CTA: blockIdx of ppo_fwd_delta_kernel, or a slot of the persistent kernel.
template <bool STAGED>
__device__ __forceinline__ void fwd_delta_block(const PpoArgs& a, int bx, int net, int64_t step, float* smem) {
  const MlpDesc& d = net ? a.critic : a.actor;
  unsigned long long* tr = (a.trace && bx == 0 && threadIdx.x == 0) ? a.trace + 16 * net : nullptr;
  int ntr = 0;
  auto mark = [&]() {
    if (tr && ntr < 16) tr[ntr++] = clock64();
  };
  mark();
  Smem s;
  carve(a, net, smem, &s);
  const int R = a.R;
  const int ldx = (a.S + 3) & ~3;
  const int A = a.A, ldA = (A + 3) & ~3;
  const int q0 = bx * R;
  const int nrows = min(R, a.mb - q0);
  const double mean = a.advstat[0], denom = a.advstat[1];
  if (STAGED) stage_weights(a, d, s.w);
  mark();
  // the gather below overlaps with the weight copies in flight; waited before the forward
  // Per-layer pointers are recomputed from the shared-memory base instead of being kept in
  // runtime-indexed arrays: an array of pointers lands in local memory and every access
  // through it becomes a generic (LD/ST) instead of a shared (LDS/STS) access.
  const int R8 = (R + 7) & ~7;
  auto h_of = [&](int l) -> float* {
    float* p = s.h0;
    for (int i = 0; i < l; ++i) p += (size_t)R8 * ((d.dims[i + 1] + 3) & ~3);
    return p;
  };
  auto ldh_of = [&](int l) { return (d.dims[l + 1] + 3) & ~3; };
  auto w_of = [&](int l) -> const float* {
    if (!STAGED) return a.params + d.off[l];
    float* p = s.w;
    for (int i = 0; i < l; ++i) p += (size_t)d.dims[i] * (d.dims[i + 1] + 1);
    return p;
  };
  auto ldw_of = [&](int l) { return STAGED ? d.dims[l + 1] + 1 : d.dims[l + 1]; };
  auto b_of = [&](int l) { return a.params + d.off[l] + (size_t)d.dims[l] * d.dims[l + 1]; };
  // ---- gather (gather_minibatch ppo.hpp:83-103): a warp per row, every load of a row in flight ----
  for (int r = threadIdx.x / 32; r < nrows; r += blockDim.x / 32) {
    const uint32_t i = mb_row(a, step, (uint32_t)(q0 + r));
    const int lane = threadIdx.x & 31;
    const float* fr = nullptr;
    if (a.obs_mode == 1) fr = a.feat + (size_t)a.row[i / a.N] * (a.S - a.Sp);
    float xv[kGatherUnroll];
#pragma unroll
    for (int u = 0; u < kGatherUnroll; ++u) {
      const int c = lane + 32 * u;
      float v = 0.0f;
      if (c < a.S) {
        if (a.obs_mode == 1)
          v = (c < a.Sp) ? a.obs[(size_t)i * a.Sp + c] : fr[c - a.Sp];
        else
          v = a.obs[(size_t)i * a.S + c];
      }
      xv[u] = v;
    }
    for (int c = lane + 32 * kGatherUnroll; c < a.S; c += 32)  // wide observations
      s.x[r * ldx + c] = (a.obs_mode == 1) ? ((c < a.Sp) ? a.obs[(size_t)i * a.Sp + c] : fr[c - a.Sp])
                                           : a.obs[(size_t)i * a.S + c];
    float act = 0.f, lp0 = 0.f, advv = 0.f, retv = 0.f;
    if (net == 0) {
      act = (lane < A) ? a.act[(size_t)i * A + lane] : 0.0f;
      if (lane == 0) {
        lp0 = a.logp[i];
        advv = a.adv[i];
      }
    } else if (lane == 0) {
      retv = a.ret[i];
    }
#pragma unroll
    for (int u = 0; u < kGatherUnroll; ++u)
      if (lane + 32 * u < a.S) s.x[r * ldx + lane + 32 * u] = xv[u];
    if (net == 0) {
      if (lane < A) s.actn[r * ldA + lane] = act;
      for (int c = lane + 32; c < A; c += 32) s.actn[r * ldA + c] = a.act[(size_t)i * A + c];
    }
    if (lane == 0) {
      s.misc[r * 4 + 0] = lp0;
      s.misc[r * 4 + 1] = (float)(((double)advv - mean) / denom);
      s.misc[r * 4 + 2] = retv;
    }
  }
  mark();
  if (STAGED) stage_wait();
  __syncthreads();
  mark();
  // ---- forward with caches (mlp_forward nn.hpp:63-85) ----
  {  // one compact instantiation (RB = 2 rows per thread per pass): the generic dispatcher's
     // four RB variants x2 activations overflow the instruction cache in this kernel
    const float* in = s.x;
    int ldi = ldx;
#pragma unroll 1
    for (int l = 0; l < d.nl; ++l) {
      const int out = d.dims[l + 1];
      int TJ = 32;
      while (TJ < out && TJ < (int)blockDim.x) TJ <<= 1;
      if (l + 1 < d.nl)
        linear_tile_rb<true, 2>(w_of(l), ldw_of(l), b_of(l), d.dims[l], out, in, ldi, h_of(l), ldh_of(l), nrows, TJ);
      else
        linear_tile_rb<false, 2>(w_of(l), ldw_of(l), b_of(l), d.dims[l], out, in, ldi, h_of(l), ldh_of(l), nrows, TJ);
      mark();
      __syncthreads();
      in = h_of(l);
      ldi = ldh_of(l);
    }
  }
  mark();
  // layer inputs for the gradient GEMMs: the observation (actor CTAs) and every hidden activation
  if (net == 0) store_rows_g(a.slab + a.hin_off[0][0], a.S, s.x, ldx, nrows, q0);
  for (int l = 1; l < d.nl; ++l) store_rows_g(a.slab + a.hin_off[net][l], d.dims[l], h_of(l - 1), ldh_of(l - 1), nrows, q0);
  mark();
  // ---- per-row losses and head gradients (ppo.hpp:128-167) ----
  const float inv_n = 1.0f / (float)a.mb;
  float* head = h_of(d.nl - 1);
  const int ldm = ldh_of(d.nl - 1);
  if (net == 0) {
    const float* log_std = a.params + a.log_std_off;
    const int Q = (A + 3) / 4;
    int L = 1;
    while (L < Q && L < 32) L <<= 1;
    const int rpp = blockDim.x / L;
    const int lir = threadIdx.x % L;
    const int rmax = ((nrows + rpp - 1) / rpp) * rpp;
    for (int r = threadIdx.x / L; r < rmax; r += rpp) {
      const bool on = r < nrows;
      float lpv = 0.0f;
      if (on)
        for (int dd = lir; dd < A; dd += L) {
          const float ls = log_std[dd];
          const float z = (s.actn[r * ldA + dd] - head[r * ldm + dd]) * expf(-ls);  // (a - mu) / sigma
          lpv += (-0.5f * kLogTwoPiF - ls) - 0.5f * z * z;
        }
      for (int o = L / 2; o > 0; o >>= 1) lpv += __shfl_xor_sync(0xffffffffu, lpv, o, L);
      if (on) {
        const float ratio = expf(lpv - s.misc[r * 4 + 0]);
        const float adv = s.misc[r * 4 + 1];
        const float surr1 = ratio * adv;
        const float lo = (float)(1.0 - a.clip), hi = (float)(1.0 + a.clip);
        const float clipped = (ratio < lo) ? lo : ((hi < ratio) ? hi : ratio);  // std::clamp
        const float surr2 = clipped * adv;
        const float dl_dlp = (surr1 <= surr2) ? -adv * ratio * inv_n : 0.0f;  // ppo.hpp:146
        for (int dd = lir; dd < A; dd += L) {
          const float ls = log_std[dd];
          const float isig = expf(-ls);
          const float z = (s.actn[r * ldA + dd] - head[r * ldm + dd]) * isig;
          head[r * ldm + dd] = dl_dlp * (z * isig);  // dmean = dL/dlp * z / sigma, in place
          s.tmp[r * ldA + dd] = dl_dlp * (z * z - 1.0f);
        }
        if (lir == 0) s.loss[r] = -((surr2 < surr1) ? surr2 : surr1) * inv_n;  // std::min (NaN-propagating)
      }
    }
  } else {
    for (int r = threadIdx.x; r < nrows; r += blockDim.x) {
      const float err = head[r * ldm] - s.misc[r * 4 + 2];
      s.loss[r] = err * err * inv_n;
      head[r * ldm] = (float)a.vf * 2.0f * err * inv_n;  // dV, in place
    }
  }
  __syncthreads();
  mark();
  // head delta, log_std terms (actor) and this net's per-row loss column
  store_rows_g(a.slab + a.del_off[net][d.nl - 1], d.dims[d.nl], head, ldm, nrows, q0);
  if (net == 0) store_rows_g(a.slab + a.ls_off, A, s.tmp, ldA, nrows, q0);
  for (int r = threadIdx.x; r < nrows; r += blockDim.x) a.slab[a.loss_off + (size_t)(q0 + r) * 2 + net] = s.loss[r];
  const int ldp = a.ldw > ldA ? a.ldw : ldA;
  mark();
  // ---- backward deltas (mlp_backward_accumulate nn.hpp:105-132, the matmul_nt half) ----
  const float* delta = head;
  int ldd = ldm;
  for (int l = d.nl - 1; l >= 1; --l) {
    const int in = d.dims[l], out = d.dims[l + 1];
    float* dp = (delta == s.d0) ? s.d1 : s.d0;
    delta_prev_tile(delta, ldd, out, w_of(l), ldw_of(l), in, h_of(l - 1), ldh_of(l - 1), dp, ldp, nrows);
    __syncthreads();
    mark();
    store_rows_g(a.slab + a.del_off[net][l - 1], in, dp, ldp, nrows, q0);
    delta = dp;
    ldd = ldp;
    mark();
  }
}

// MODE: 0 weights read from L2, 1 staged (fwd_delta_block), 2 rows-of-8 path (fwd_delta_r8)
template <int MODE>
__device__ __forceinline__ void fwd_delta_any(const PpoArgs& a, int bx, int net, int64_t step, float* smem,
                                              uint64_t* mbar = nullptr, uint32_t* mphase = nullptr,
                                              const uint2* rows = nullptr) {
  if (MODE == 2)
    fwd_delta_r8(a, bx, net, step, smem, mbar, mphase, rows);
  else
    fwd_delta_block<MODE == 1>(a, bx, net, step, smem);
}

template <int MODE>
__global__ void __launch_bounds__(kPpoThreads) ppo_fwd_delta_kernel(PpoArgs a) {
  if (a.status[0] != 0) return;
  extern __shared__ __align__(16) float smem[];
  fwd_delta_any<MODE>(a, blockIdx.x, blockIdx.y, *a.step, smem);
}

// ---- ppo_grad: output-parallel dW / db / dlog_std, fixed-order sums, step gate ----
constexpr int kGT = 64;        // output tile (k rows x j cols of [W; b])
constexpr int kGChunk = 64;    // rows per sub-chunk of a split (one float4 load round)
constexpr int kGLd = kGT + 4;  // smem row stride (float4-aligned)
constexpr int kMaxSplits = 32;  // row splits per tile (each split loops over kGChunk-row sub-chunks)
constexpr int kGRows = 16;      // minimum rows per split

struct GradArgs {
  const float* slab;
  int hin_off[2][kMaxLayers], del_off[2][kMaxLayers], ls_off, loss_off;
  MlpDesc net[2];
  int mb, RS, P, Pext, log_std_off, A;
  const int4* tiles;  // {net, layer (-1: log_std + losses), k0, j0}
  int ntiles;
  float* partial;     // [RS][Pext]
  float* grads;
  int32_t* tickets;   // [0] ppo_sum completed-CTA counter, [1] gradient non-finite flag
  double ent;
  const float* params;
  int32_t* status;
  int64_t* t;
  int64_t* step;
  double* stats;
  int apply;
  unsigned long long* trace;  // debug (PRB_PPO_TRACE): [grid][8] globaltimer marks, else null
  // Adam (adam_step nn.hpp:164-182), applied by ppo_sum_adam once the gate is known
  float* p_rw;
  float* m;
  float* v;
  float lr, eps;
  double b1, b2;
};

__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// virtual CTA vb = tile * RS + split (blockIdx.x of ppo_grad_kernel, or a persistent slot)
__device__ __forceinline__ void grad_block(const GradArgs& g, int vb, float* gsm, unsigned long long* btr = nullptr) {
  float* As = gsm;
  float* Bs = gsm + kGChunk * kGLd;
  const int tile = vb / g.RS, split = vb % g.RS;
  const int4 td = g.tiles[tile];
  const int per = (g.mb + g.RS - 1) / g.RS;  // rows of this split, processed in kGChunk sub-chunks
  const int rbeg = split * per, rend = min(g.mb, rbeg + per);
  const int tid = threadIdx.x;
  float* part = g.partial + (size_t)split * g.Pext;
  if (td.y >= 0) {
    const MlpDesc& d = g.net[td.x];
    const int l = td.y, in = d.dims[l], out = d.dims[l + 1], k0 = td.z, j0 = td.w;
    const float* H = g.slab + g.hin_off[td.x][l];
    const float* D = g.slab + g.del_off[td.x][l];
    // thread = 4 k x 4 j outputs; warp w owns columns j0 + 8w .. 8w+7, so warps past `out` skip the math
    const int tk = tid & 15, tj = tid >> 4;
    const bool active = j0 + 8 * (tid >> 5) < out;
    const bool with_bias = (k0 == 0);  // the k0 = 0 tile also sums delta's columns (the bias row)
    float acc[4][4], bsum[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) acc[i][j] = 0.0f;
    for (int r0 = rbeg; r0 < rend; r0 += kGChunk) {
      const int nr = min(kGChunk, rend - r0);
      __syncthreads();  // previous sub-chunk consumed
      // float4 columns (slab rows are padded to a multiple of 4 floats, the padding zero):
      // 16 float4 per 64-wide tile row, 16 rows per pass, every load of the sub-chunk in
      // flight before the first store
      const int c4 = tid & 15, rr = tid >> 4;
      const int k = k0 + 4 * c4, j = j0 + 4 * c4;
      const int ldh = (in + 3) & ~3, ldd = (out + 3) & ~3;
      float4 av[kGChunk / 16], bv[kGChunk / 16];
#pragma unroll
      for (int u = 0; u < kGChunk / 16; ++u) {
        const int r = rr + 16 * u;
        const size_t row = (size_t)(r0 + r);
        av[u] = (r < nr && k < in) ? *reinterpret_cast<const float4*>(H + row * ldh + k) : make_float4(0.f, 0.f, 0.f, 0.f);
        bv[u] = (r < nr && j < out) ? *reinterpret_cast<const float4*>(D + row * ldd + j) : make_float4(0.f, 0.f, 0.f, 0.f);
      }
#pragma unroll
      for (int u = 0; u < kGChunk / 16; ++u) {
        const int r = rr + 16 * u;
        if (r < nr) {
          *reinterpret_cast<float4*>(As + r * kGLd + 4 * c4) = av[u];
          *reinterpret_cast<float4*>(Bs + r * kGLd + 4 * c4) = bv[u];
        }
      }
      __syncthreads();
      if (btr) btr[0] = gtime();
      if (active) {
#pragma unroll 4
        for (int r = 0; r < nr; ++r) {
          const float4 av = *reinterpret_cast<const float4*>(As + r * kGLd + 4 * tk);
          const float4 bv = *reinterpret_cast<const float4*>(Bs + r * kGLd + 4 * tj);
          const float ak[4] = {av.x, av.y, av.z, av.w}, bj[4] = {bv.x, bv.y, bv.z, bv.w};
#pragma unroll
          for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 4; j += 2) tc::fma2(acc[i][j], acc[i][j + 1], ak[i], bj[j], bj[j + 1]);
          if (with_bias) {
#pragma unroll
            for (int j = 0; j < 4; ++j) bsum[j] += bj[j];
          }
        }
      }
    }
    if (btr) btr[1] = gtime();
    // the tile through shared memory, then row segments stored by whole warps (coalesced: a
    // thread's 4x4 block spans 4 rows, so direct stores would touch 16 rows per instruction)
    __syncthreads();  // As/Bs free
    if (active) {
#pragma unroll
      for (int i = 0; i < 4; ++i)
        *reinterpret_cast<float4*>(As + (4 * tk + i) * kGLd + 4 * tj) =
            make_float4(acc[i][0], acc[i][1], acc[i][2], acc[i][3]);
      if (with_bias && tk == 0) *reinterpret_cast<float4*>(Bs + 4 * tj) = make_float4(bsum[0], bsum[1], bsum[2], bsum[3]);
    }
    __syncthreads();
    const int nk = min(kGT, in - k0), nj = min(kGT, out - j0);
    const int lane = tid & 31;
    float* pw = part + d.off[l] + j0;
    for (int kr = tid >> 5; kr < nk; kr += 8) {
      float* rowp = pw + (size_t)(k0 + kr) * out;
      if (lane < nj) rowp[lane] = As[kr * kGLd + lane];
      if (lane + 32 < nj) rowp[lane + 32] = As[kr * kGLd + lane + 32];
    }
    if (with_bias && tid < 64 && tid < nj) pw[(size_t)in * out + tid] = Bs[tid];
  } else {  // log_std terms and the two loss sums over this split's rows
    const float* LS = g.slab + g.ls_off;
    const float* LO = g.slab + g.loss_off;
    for (int c = tid; c < g.A + 2; c += 256) {
      const float* src = (c < g.A) ? LS + c : LO + (c - g.A);
      const int ld = (c < g.A) ? ((g.A + 3) & ~3) : 2;  // log_std rows padded like every slab array
      float acc = 0.0f;
      for (int r = rbeg; r < rend; r += 16) {  // 16 loads in flight, summed in row order
        float v[16];
#pragma unroll
        for (int u = 0; u < 16; ++u) v[u] = (r + u < rend) ? src[(size_t)(r + u) * ld] : 0.0f;
#pragma unroll
        for (int u = 0; u < 16; ++u)
          if (r + u < rend) acc += v[u];
      }
      part[c < g.A ? g.log_std_off + c : g.P + (c - g.A)] = acc;
    }
  }
}

__global__ void __launch_bounds__(256) ppo_grad_kernel(GradArgs g) {
  unsigned long long* tr = (g.trace && threadIdx.x == 0) ? g.trace + (size_t)blockIdx.x * 8 : nullptr;
  if (tr) tr[0] = gtime();
  if (g.status[0] != 0) return;
  extern __shared__ __align__(16) float gsm[];
  grad_block(g, blockIdx.x, gsm);
  if (tr) tr[1] = gtime();
}

// ---- ppo_sum: grads[p] = sum of the split partials in split order (+ entropy term for
// log_std), non-finite flag; the last CTA evaluates the step's gate (losses first, then
// gradients: the reference order) and advances t / the minibatch counter ----
// ---- ppo_sum_adam: grads[p] = sum of the split partials in split order (+ entropy term
// for log_std) and the non-finite flag; the last CTA to finish evaluates the step's gate
// (losses first, then gradients: the reference order), advances t / the minibatch counter
// and releases the others, which then apply Adam to their parameter range (skipped when
// the gate failed, so a rejected step leaves params/m/v/t untouched, nn.hpp:169-171).
// Launched cooperatively (every CTA resident), grid-stride over the parameters.
// adam_step (nn.hpp:164-182) for one fp32 parameter with every rounding explicit: the device
// compiler's FMA contraction choices can differ between kernels, and the persistent and the
// per-kernel updates must agree bit for bit
__device__ __forceinline__ void adam_param(float b1, float b2, float omb1, float omb2, float lr, float eps, float ibc1,
                                           float ibc2, float g, float& m, float& v, float& w) {
  m = __fmaf_rn(b1, m, __fmul_rn(omb1, g));
  v = __fmaf_rn(b2, v, __fmul_rn(__fmul_rn(omb2, g), g));
  w = __fsub_rn(w, __fdiv_rn(__fmul_rn(lr, __fmul_rn(m, ibc1)), __fadd_rn(__fsqrt_rn(__fmul_rn(v, ibc2)), eps)));
}

__global__ void __launch_bounds__(256) ppo_sum_adam_kernel(GradArgs g) {
  if (g.status[0] != 0) return;
  const int tid = threadIdx.x;
  int bad = 0;
  for (int p = blockIdx.x * 256 + tid; p < g.P; p += gridDim.x * 256) {
    float v[kMaxSplits];
#pragma unroll
    for (int sp = 0; sp < kMaxSplits; ++sp) v[sp] = (sp < g.RS) ? g.partial[(size_t)sp * g.Pext + p] : 0.0f;
    float sum = 0.0f;
#pragma unroll
    for (int sp = 0; sp < kMaxSplits; ++sp)
      if (sp < g.RS) sum += v[sp];
    if (p >= g.log_std_off && p < g.log_std_off + g.A) sum -= (float)g.ent;  // ppo.hpp:157
    g.grads[p] = sum;
    bad |= !isfinite(sum);
  }
  if (__syncthreads_or(bad) && tid == 0) atomicOr(&g.tickets[1], 1);
  __threadfence();
  __shared__ int lastall;
  if (tid == 0) lastall = (atomicAdd(&g.tickets[0], 1) == (int)gridDim.x - 1);
  __syncthreads();
  if (lastall) {
    __threadfence();
    // split loss sums and log_std values loaded by the block, summed by one thread in order
    __shared__ double red[2 * kMaxSplits + 256];
    if (tid < g.RS) {
      red[tid] = g.partial[(size_t)tid * g.Pext + g.P];
      red[kMaxSplits + tid] = g.partial[(size_t)tid * g.Pext + g.P + 1];
    }
    for (int dd = tid; dd < g.A && dd < 256; dd += 256) red[2 * kMaxSplits + dd] = (double)g.params[g.log_std_off + dd];
    __syncthreads();
    if (tid == 0) {
      double pl = 0.0, vl = 0.0;
      for (int sp = 0; sp < g.RS; ++sp) {
        pl += red[sp];
        vl += red[kMaxSplits + sp];
      }
      double ent = 0.0;  // policy_entropy nn.hpp:273-277
      for (int dd = 0; dd < g.A; ++dd)
        ent += 0.5 * (1.8378770664093454836 + 1.0) +
               (dd < 256 ? red[2 * kMaxSplits + dd] : (double)g.params[g.log_std_off + dd]);
      const int gbad = atomicAdd(&g.tickets[1], 0);
      g.tickets[1] = 0;
      if (!isfinite(pl)) {
        g.status[0] = PRB_ERR_NUMERIC;
        g.status[1] = 10;
      } else if (!isfinite(vl)) {
        g.status[0] = PRB_ERR_NUMERIC;
        g.status[1] = 11;
      } else if (!isfinite(ent)) {
        g.status[0] = PRB_ERR_NUMERIC;
        g.status[1] = 12;
      } else if (gbad && g.apply) {
        g.status[0] = PRB_ERR_NUMERIC;
        g.status[1] = 1;
      } else {
        g.stats[0] += pl;
        g.stats[1] += vl;
        g.stats[2] += ent;
        g.stats[3] += 1.0;
        if (g.apply) *g.t += 1;
      }
      *g.step += 1;
      __threadfence();
      atomicExch(&g.tickets[0], 0);  // release the waiting CTAs
    }
  } else if (tid == 0) {
    while (atomicAdd(&g.tickets[0], 0) != 0) {
    }
  }
  __syncthreads();
  __threadfence();
  if (!g.apply || *(volatile int32_t*)g.status != 0) return;
  // ---- Adam on this CTA's parameters (adam_kernel's arithmetic, agent.cu) ----
  __shared__ float sb[2];
  if (tid == 0) {
    const int64_t t = *(volatile int64_t*)g.t;
    sb[0] = (float)(1.0 / (1.0 - pow(g.b1, (double)t)));
    sb[1] = (float)(1.0 / (1.0 - pow(g.b2, (double)t)));
  }
  __syncthreads();
  const float ibc1 = sb[0], ibc2 = sb[1];
  const float b1 = (float)g.b1, b2 = (float)g.b2, omb1 = (float)(1.0 - g.b1), omb2 = (float)(1.0 - g.b2);
  for (int p = blockIdx.x * 256 + tid; p < g.P; p += gridDim.x * 256) {
    float mi = g.m[p], vi = g.v[p], wi = g.p_rw[p];
    adam_param(b1, b2, omb1, omb2, g.lr, g.eps, ibc1, ibc2, g.grads[p], mi, vi, wi);
    g.m[p] = mi;
    g.v[p] = vi;
    g.p_rw[p] = wi;
  }
}

// ---- persistent update: every minibatch step of a ppo_update in ONE cooperative launch ----
// The four phases of a step are separated by grid-wide barriers instead of kernel
// boundaries (a graph of 3 launches per minibatch spent most of its time filling and
// draining the GPU between dependent kernels).  Per step:
//   A  fwd_delta_block over the (mb/R) x 2 row blocks          | barrier
//   B  grad_block over the ntiles x RS output tiles            | barrier
//   C1 split sums -> grads (+ entropy term), non-finite flag; the CTA snapshots log_std and t
//                                                              | barrier
//   C2 every CTA evaluates the same gate from the same inputs (losses first, then gradients:
//      the reference order); CTA 0 alone publishes status / stats / t; Adam on the CTA's
//      parameter range (skipped, and the loop left by every CTA, when the gate fails)
//                                                              | barrier
// The arithmetic of every phase is the per-kernel path's (same device functions, same
// reduction orders), so both paths give bit-identical parameters.
// Monotonic arrival counter: barrier i of the launch completes when the counter reaches
// (i+1) * nblocks.  Arrival is a release reduction, the wait an acquire load, so the
// writes of every CTA before the barrier are visible to every CTA after it (the
// __syncthreads on both sides extend this to the whole CTA).  No reset, no generation
// word: the last arrival's single reduction releases everyone.
__device__ __forceinline__ void grid_barrier(unsigned int* count, unsigned int& target, unsigned int nblocks) {
  target += nblocks;
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(count) : "memory");
    unsigned int v;
    unsigned long long t0 = 0;
    int polls = 0;
    do {
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(count) : "memory");
      if ((++polls & 1023) == 0) barrier_watchdog(t0);
    } while ((int)(v - target) < 0);
  }
  __syncthreads();
}

// parameter p's copy in the staged-weight image (persistent rows-of-8 update)
__device__ __forceinline__ void img_store(const PpoArgs& a, int p, float v) {
  int q = r8_img_pos(a.actor, p);
  if (q < 0) {
    q = r8_img_pos(a.critic, p);
    if (q >= 0) q += a.img_c;
  }
  if (q >= 0) a.wimg[q] = v;
}

template <int MODE>
__global__ void __launch_bounds__(kPpoThreads, 2) ppo_persistent_kernel(PpoArgs a, GradArgs g, int64_t steps,
                                                                     unsigned int* bar, int32_t* flags,
                                                                     float2* bias_tab, unsigned long long* trace) {
  extern __shared__ __align__(16) float smem[];
  __shared__ float s_ls[256];
  __shared__ double s_lsum[2 * kMaxSplits];
  __shared__ int s_lcode;
  __shared__ double s_loss[3];
  __shared__ __align__(8) uint64_t s_mbar;  // bulk staging of the weight image (MODE 2)
  const int tid = threadIdx.x;
  const bool img = MODE == 2 && a.wimg;
  uint64_t* mbar = img ? &s_mbar : nullptr;
  uint32_t mphase = 0;
  if (img) {
    if (tid == 0) tc::mbar_init(&s_mbar, 1);
    for (int p = blockIdx.x * 256 + tid; p < a.P; p += gridDim.x * 256) img_store(a, p, a.params[p]);
    asm volatile("fence.proxy.async.global;" ::: "memory");
  }
  const unsigned int nb = gridDim.x;
  unsigned int bt = 0;  // barrier target
  const int nA = (a.mb + a.R - 1) / a.R;
  const int nB = g.ntiles * g.RS;
  const float b1 = (float)g.b1, b2 = (float)g.b2, omb1 = (float)(1.0 - g.b1), omb2 = (float)(1.0 - g.b2);
  // Adam bias corrections of every step, computed once up front (adam_kernel's fp64 pow):
  // step st runs with t = t0 + st + 1 (a failed gate ends the update, so t never skips)
  {
    const int64_t t0 = *g.t;
    for (int64_t i = (int64_t)blockIdx.x * 256 + tid; i < steps; i += (int64_t)nb * 256) {
      const double t = (double)(t0 + i + 1);
      bias_tab[i] = make_float2((float)(1.0 / (1.0 - pow(g.b1, t))), (float)(1.0 / (1.0 - pow(g.b2, t))));
    }
  }
  grid_barrier(bar, bt, nb);
  // PRB_PPO_TRACE: globaltimer stamps of step 4 per CTA (phase ends and barrier exits)
  unsigned long long* tr = (trace && tid == 0) ? trace + (size_t)blockIdx.x * 16 : nullptr;
  const int p0 = blockIdx.x * 256 + tid;  // this thread's first parameter (its Adam update is kept in registers)
  const bool spec = (int64_t)nb * 256 >= g.P && !a.nospec;  // every parameter has its own thread
  const bool pf = MODE == 2 && a.rtab && (int)nb > 2 * nA;   // CTAs without a row block exist
  for (int64_t st = 0; st < steps; ++st) {
    const bool mk = tr && st == (steps > 4 ? 4 : 0);
    if (mk) tr[0] = gtime();
    // ---- A: forward + head gradients + backward deltas, row-parallel; the CTAs without a row
    // block resolve the next step's minibatch rows (Feistel permutation + feature row) ----
    if (pf && (int)blockIdx.x >= 2 * nA && st + 1 < steps) {
      uint2* t = a.rtab + ((st + 1) & 1) * a.mb;
      for (int q = ((int)blockIdx.x - 2 * nA) * 256 + tid; q < a.mb; q += ((int)nb - 2 * nA) * 256) {
        const uint32_t i = mb_row(a, st + 1, (uint32_t)q);
        t[q] = make_uint2(i, a.obs_mode == 1 ? (uint32_t)a.row[i / a.N] : 0u);
      }
    }
    const uint2* rows = (pf && st > 0) ? a.rtab + (st & 1) * a.mb : nullptr;
    for (int vb = blockIdx.x; vb < 2 * nA; vb += nb) {
      fwd_delta_any<MODE>(a, vb % nA, vb / nA, st, smem, mbar, &mphase, rows);
      __syncthreads();
    }
    if (mk) tr[1] = gtime();
    grid_barrier(bar, bt, nb);
    if (mk) tr[2] = gtime();
    // ---- B: dW / db / log_std / loss split partials, output-parallel ----
    for (int vb = blockIdx.x; vb < nB; vb += nb) {
      grad_block(g, vb, smem, (mk && vb == (int)blockIdx.x) ? tr + 10 : nullptr);
      __syncthreads();
    }
    if (mk) tr[3] = gtime();
    for (int dd = tid; dd < g.A; dd += 256) s_ls[dd] = g.params[g.log_std_off + dd];  // before any Adam write
    grid_barrier(bar, bt, nb);
    if (mk) tr[4] = gtime();
    // ---- C1: split sums in split order (ppo_sum_adam_kernel's arithmetic), the loss half of
    // the gate, and this thread's first Adam update computed speculatively ----
    const float2 bc = bias_tab[st];
    float np0 = 0.f, nm0 = 0.f, nv0 = 0.f;
    float m0 = 0.f, v0 = 0.f, w0 = 0.f;
    if (p0 < g.P) {  // issued with the partial loads below
      m0 = g.m[p0];
      v0 = g.v[p0];
      w0 = g.p_rw[p0];
    }
    if (tid >= 32 && tid < 32 + g.RS) {  // loss split sums (gate inputs)
      s_lsum[tid - 32] = (double)g.partial[(size_t)(tid - 32) * g.Pext + g.P];
      s_lsum[kMaxSplits + tid - 32] = (double)g.partial[(size_t)(tid - 32) * g.Pext + g.P + 1];
    }
    int bad = 0;
    for (int p = p0; p < g.P; p += nb * 256) {
      float v[kMaxSplits];
#pragma unroll
      for (int sp = 0; sp < kMaxSplits; ++sp) v[sp] = (sp < g.RS) ? g.partial[(size_t)sp * g.Pext + p] : 0.0f;
      float sum = 0.0f;
#pragma unroll
      for (int sp = 0; sp < kMaxSplits; ++sp)
        if (sp < g.RS) sum += v[sp];
      if (p >= g.log_std_off && p < g.log_std_off + g.A) sum -= (float)g.ent;  // ppo.hpp:157
      bad |= !isfinite(sum);
      if (p == p0) {
        nm0 = m0;
        nv0 = v0;
        np0 = w0;
        adam_param(b1, b2, omb1, omb2, g.lr, g.eps, bc.x, bc.y, sum, nm0, nv0, np0);
      } else {
        g.grads[p] = sum;
      }
    }
    if (__syncthreads_or(bad) && tid == 0) atomicOr(&flags[st & 1], 1);
    if (tid == 0) {  // losses first (the reference order); gradients after the barrier
      double pl = 0.0, vl = 0.0;
      for (int sp = 0; sp < g.RS; ++sp) {
        pl += s_lsum[sp];
        vl += s_lsum[kMaxSplits + sp];
      }
      double ent = 0.0;  // policy_entropy nn.hpp:273-277
      for (int dd = 0; dd < g.A; ++dd) ent += 0.5 * (1.8378770664093454836 + 1.0) + (double)s_ls[dd];
      s_lcode = !isfinite(pl) ? 10 : (!isfinite(vl) ? 11 : (!isfinite(ent) ? 12 : 0));
      s_loss[0] = pl;
      s_loss[1] = vl;
      s_loss[2] = ent;
    }
    // one parameter per thread: the Adam update is stored now and undone from the registers
    // if the gate (known after the barrier) fails -- one grid barrier per step fewer
    if (spec && p0 < g.P) {
      g.m[p0] = nm0;
      g.v[p0] = nv0;
      g.p_rw[p0] = np0;
      if (img) img_store(a, p0, np0);
    }
    if (spec && img) asm volatile("fence.proxy.async.global;" ::: "memory");
    if (mk) tr[5] = gtime();
    grid_barrier(bar, bt, nb);
    if (mk) tr[6] = gtime();
    // ---- C2: the gate (identical in every CTA), then Adam: the first parameter from
    // registers, any further ones (wide nets) recomputed from grads ----
    const int code = s_lcode ? s_lcode : (*(volatile int32_t*)&flags[st & 1] ? 1 : 0);
    if (blockIdx.x == 0 && tid == 0) {
      if (code) {
        g.status[0] = PRB_ERR_NUMERIC;
        g.status[1] = code;
      } else {
        g.stats[0] += s_loss[0];
        g.stats[1] += s_loss[1];
        g.stats[2] += s_loss[2];
        g.stats[3] += 1.0;
        *g.t += 1;
      }
      *g.step += 1;
      flags[(st + 1) & 1] = 0;  // next step's flag: last read before the previous barrier
    }
    if (code) {  // identical decision in every CTA
      if (spec && p0 < g.P) {  // nn.hpp:169-171: a rejected step leaves params, m and v untouched
        g.m[p0] = m0;
        g.v[p0] = v0;
        g.p_rw[p0] = w0;
        if (img) img_store(a, p0, w0);
      }
      break;
    }
    if (spec) {
      if (mk) tr[7] = tr[8] = gtime();
      continue;
    }
    if (p0 < g.P) {
      g.m[p0] = nm0;
      g.v[p0] = nv0;
      g.p_rw[p0] = np0;
      if (img) img_store(a, p0, np0);
    }
    for (int p = p0 + nb * 256; p < g.P; p += nb * 256) {
      float mi = g.m[p], vi = g.v[p], np = g.p_rw[p];
      adam_param(b1, b2, omb1, omb2, g.lr, g.eps, bc.x, bc.y, g.grads[p], mi, vi, np);
      g.m[p] = mi;
      g.v[p] = vi;
      g.p_rw[p] = np;
      if (img) img_store(a, p, np);
    }
    if (img) asm volatile("fence.proxy.async.global;" ::: "memory");  // image -> next step's bulk copies
    if (mk) tr[7] = gtime();
    grid_barrier(bar, bt, nb);
    if (mk) tr[8] = gtime();
  }
}

struct PpoWorkspace {
  DevBuf<float> partial;   // [RS][Pext] split partials of the gradient GEMMs
  DevBuf<float> slab;      // per-row layer inputs / deltas of one minibatch
  DevBuf<int4> tiles;      // ppo_grad tile list
  DevBuf<int32_t> tickets; // [ntiles] split tickets, completed-tile counter, gradient flag
  int ntiles = 0, RS = 1;
  DevBuf<int64_t> step;
  DevBuf<double> stats;
  DevBuf<uint32_t> perm;
  DevBuf<unsigned long long> trace;  // PRB_PPO_TRACE
  DevBuf<int32_t> bar;               // persistent update: grid barrier + non-finite flags
  DevBuf<float2> bias;               // persistent update: Adam bias corrections per step
  DevBuf<unsigned long long> ptrace; // PRB_PPO_TRACE of the persistent update: [grid][10]
  DevBuf<float> wimg;                // persistent rows-of-8 update: staged-layout weight image
  DevBuf<uint2> rtab;                // ... and the next step's resolved minibatch rows
  // tensor-core update (ppo_tc.cu): weight image, per-CTA partial slab, stats, chain descriptor
  DevBuf<uint8_t> tc_img;
  DevBuf<float> tc_slab;
  DevBuf<double> tc_stats;
  DevBuf<uint32_t> tc_sync;
  DevBuf<PpoTcChain> tc_chain;
  DevBuf<int2> tc_pos;  // weight-image position of every parameter (for the net shape below)
  std::vector<int> tc_pos_key;
};

PpoArgs make_args(prb_agent a, prb_rollout r, const prb_ppo_config* cfg, uint64_t seed, PpoWorkspace& ws, int mb) {
  PpoArgs p{};
  p.params = a->d_params.p;
  p.actor.nl = (int)a->adims.size() - 1;
  p.critic.nl = (int)a->cdims.size() - 1;
  for (size_t i = 0; i < a->adims.size(); ++i) p.actor.dims[i] = (int)a->adims[i];
  for (size_t i = 0; i < a->cdims.size(); ++i) p.critic.dims[i] = (int)a->cdims[i];
  for (size_t i = 0; i < a->aoff.size(); ++i) p.actor.off[i] = (int)a->aoff[i];
  for (size_t i = 0; i < a->coff.size(); ++i) p.critic.off[i] = (int)a->coff[i];
  p.log_std_off = (int)a->Pa;
  p.A = (int)a->A;
  p.P = (int)a->P;
  p.Pext = (int)((a->P + 2 + 3) & ~size_t(3));
  p.obs_mode = r->obs_mode;
  p.S = (int)r->S;
  p.Sp = (int)r->Sp;
  p.K = r->K;
  p.obs = r->d_obs.p;
  p.row = r->d_row.p;
  p.feat = r->d_feat;
  p.act = r->d_act.p;
  p.logp = r->d_logp.p;
  p.adv = r->d_adv.p;
  p.ret = r->d_ret.p;
  p.advstat = r->d_advstat.p;
  p.N = (uint32_t)r->N;
  p.seed = seed;
  p.n = (uint32_t)(r->N * r->H);
  p.mb = mb;
  p.nmb = (uint32_t)(p.n / (uint32_t)mb);
  int bits = 2;
  while (((uint64_t)1 << bits) < p.n) ++bits;
  if (bits & 1) ++bits;
  p.bits = bits;
  p.clip = cfg->clip_eps;
  p.ent = cfg->entropy_coef;
  p.vf = cfg->value_coef;
  p.status = a->d_status.p;
  int maxw = 4;
  for (size_t h : a->hidden) maxw = std::max<int>(maxw, (int)h);
  p.ldw = (maxw + 3) & ~3;
  // rows per CTA: as many CTAs as possible while every CTA keeps >= 8 rows
  p.R = 8;
  while (p.R < 64 && (size_t)(mb / (p.R * 2)) >= (size_t)a->ctx->num_sms) p.R *= 2;
  if (const char* rv = debug_env("PRB_PPO_R")) p.R = std::max(8, std::min(64, atoi(rv)));  // A/B knob
  p.stage = 1;
  p.r8 = 0;
  {  // rows-of-8 path: 8-row blocks, every layer output <= 64 wide, A <= 32
    bool ok = (p.R == 8) && p.A <= 32 && !(debug_env("PRB_PPO_R8") && atoi(debug_env("PRB_PPO_R8")) == 0);
    for (int l = 0; l < p.actor.nl; ++l) ok = ok && p.actor.dims[l + 1] <= 64;
    for (int l = 0; l < p.critic.nl; ++l) ok = ok && p.critic.dims[l + 1] <= 64;
    if (ok) {
      p.r8 = 1;
      if (carve_max(p) > kSmemBudget) p.r8 = 0;
    }
  }
  if (carve_max(p) > kSmemBudget) p.stage = 0;  // wide nets: weights stay in L2
  while (p.R > 8 && carve_max(p) > kSmemBudget) p.R /= 2;
  PRB_REQUIRE(carve_max(p) <= kSmemBudget, PRB_ERR_CONFIG, "ppo: network too wide for the SIMT tile");
  // per-row slab: observation, hidden activations (layer inputs) and deltas of both nets
  size_t off = 0;
  auto take = [&](size_t w) {
    const size_t o = off;
    off += ((size_t)mb * w + 3) & ~size_t(3);
    PRB_REQUIRE(off < ((size_t)1 << 31), PRB_ERR_CONFIG, "ppo: minibatch slab too large");
    return (int)o;
  };
  auto r4 = [](size_t w) { return (w + 3) & ~size_t(3); };  // float4-aligned rows for ppo_grad's loads
  p.hin_off[0][0] = p.hin_off[1][0] = take(r4((size_t)p.S));
  for (int net = 0; net < 2; ++net) {
    const MlpDesc& d = net ? p.critic : p.actor;
    for (int l = 1; l < d.nl; ++l) p.hin_off[net][l] = take(r4((size_t)d.dims[l]));
    for (int l = 0; l < d.nl; ++l) p.del_off[net][l] = take(r4((size_t)d.dims[l + 1]));
  }
  p.ls_off = take(r4((size_t)p.A));
  p.loss_off = take(r4(2));
  ws.slab.ensure(off);
  PRB_CUDA(cudaMemsetAsync(ws.slab.p, 0, ws.slab.bytes(), a->ctx->stream));  // row padding stays zero
  p.slab = ws.slab.p;
  // gradient tiles: every [W_l; b_l] of both nets in 64x64 output tiles, plus log_std + losses
  std::vector<int4> tiles;
  for (int net = 0; net < 2; ++net) {
    const MlpDesc& d = net ? p.critic : p.actor;
    for (int l = 0; l < d.nl; ++l)
      for (int k0 = 0; k0 < d.dims[l]; k0 += kGT)
        for (int j0 = 0; j0 < d.dims[l + 1]; j0 += kGT) tiles.push_back(make_int4(net, l, k0, j0));
  }
  tiles.push_back(make_int4(0, -1, 0, 0));
  ws.ntiles = (int)tiles.size();
  // splits: enough (tile, split) items to give every SM two of them (one wave of the persistent
  // grid), each split keeping >= kGRows rows
  ws.RS = std::max(1, std::min({kMaxSplits, (mb + kGRows - 1) / kGRows, 2 * a->ctx->num_sms / ws.ntiles}));
  ws.tiles.ensure(tiles.size());
  // every setup copy/memset on the stream the kernels run on (the context stream is
  // non-blocking: legacy-stream cudaMemset/cudaMemcpy would not be ordered with them)
  PRB_CUDA(cudaMemcpyAsync(ws.tiles.p, tiles.data(), tiles.size() * sizeof(int4), cudaMemcpyHostToDevice,
                           a->ctx->stream));
  ws.tickets.ensure(2);  // [0] completed-CTA counter of ppo_sum, [1] gradient non-finite flag
  if (debug_env("PRB_PPO_TRACE")) {
    ws.trace.alloc((size_t)ws.ntiles * ws.RS * 8 + 32);
    PRB_CUDA(cudaMemsetAsync(ws.trace.p, 0, ws.trace.bytes(), a->ctx->stream));
  }
  PRB_CUDA(cudaMemsetAsync(ws.tickets.p, 0, ws.tickets.bytes(), a->ctx->stream));
  ws.partial.ensure((size_t)ws.RS * p.Pext);
  if (!ws.step.p) ws.step.alloc(1);
  if (!ws.stats.p) ws.stats.alloc(4);
  p.step = ws.step.p;
  return p;
}

GradArgs make_grad_args(const PpoArgs& p, prb_agent a, PpoWorkspace& ws, double ent, int apply) {
  GradArgs g;
  g.slab = p.slab;
  std::memcpy(g.hin_off, p.hin_off, sizeof(g.hin_off));
  std::memcpy(g.del_off, p.del_off, sizeof(g.del_off));
  g.ls_off = p.ls_off;
  g.loss_off = p.loss_off;
  g.net[0] = p.actor;
  g.net[1] = p.critic;
  g.mb = p.mb;
  g.RS = ws.RS;
  g.P = p.P;
  g.Pext = p.Pext;
  g.log_std_off = p.log_std_off;
  g.A = p.A;
  g.tiles = ws.tiles.p;
  g.ntiles = ws.ntiles;
  g.partial = ws.partial.p;
  g.grads = a->d_grads.p;
  g.tickets = ws.tickets.p;
  g.ent = ent;
  g.params = p.params;
  g.status = a->d_status.p;
  g.t = a->d_t.p;
  g.step = ws.step.p;
  g.stats = ws.stats.p;
  g.apply = apply;
  g.trace = ws.trace.p;
  g.p_rw = a->d_params.p;
  g.m = a->d_m.p;
  g.v = a->d_v.p;
  g.lr = (float)a->lr;
  g.eps = (float)a->eps;
  g.b1 = a->beta1;
  g.b2 = a->beta2;
  return g;
}

void launch_coop(const void* fn, int grid, size_t smem, cudaStream_t s, void** args) {
  PRB_CUDA(cudaLaunchCooperativeKernel(fn, dim3(grid), dim3(256), args, smem, s));
}

void launch_step(const PpoArgs& p, prb_agent a, PpoWorkspace& ws, double ent, int apply, cudaStream_t s) {
  const dim3 grid((p.mb + p.R - 1) / p.R, 2);
  PpoArgs pt = p;
  pt.trace = ws.trace.p ? ws.trace.p + (size_t)ws.ntiles * ws.RS * 8 : nullptr;
  const size_t smem = carve_max(p);
  // steps run inside CUDA graphs: no event scopes
  if (p.r8)
    ppo_fwd_delta_kernel<2><<<grid, kPpoThreads, smem, s>>>(pt);
  else if (p.stage)
    ppo_fwd_delta_kernel<1><<<grid, kPpoThreads, smem, s>>>(pt);
  else
    ppo_fwd_delta_kernel<0><<<grid, kPpoThreads, smem, s>>>(pt);
  GradArgs g = make_grad_args(p, a, ws, ent, apply);
  ppo_grad_kernel<<<ws.ntiles * ws.RS, 256, 2 * kGChunk * kGLd * sizeof(float), s>>>(g);
  int occ = 0;
  PRB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, ppo_sum_adam_kernel, 256, 0));
  occ = std::max(occ, 1);
  const int sgrid = std::min((p.P + 255) / 256, a->ctx->num_sms * occ);
  // cooperative: every CTA resident (the CTAs wait for the last one's gate)
  void* args[] = {&g};
  launch_coop((const void*)ppo_sum_adam_kernel, sgrid, 0, s, args);
}

size_t persistent_smem(const PpoArgs& p) {
  return std::max(carve_max(p), (size_t)(2 * kGChunk * kGLd * sizeof(float)));
}

// Grid of the persistent update (0: not launchable -> per-kernel path).
int persistent_grid(const PpoArgs& p, prb_agent a, const PpoWorkspace& ws) {
  if (p.A > 256 || debug_option(PRB_OPT_PPO_PER_KERNEL)) return 0;  // tests: force the per-kernel path
  const size_t smem = persistent_smem(p);
  int occ = 0;
  const void* fn = p.r8 ? (const void*)ppo_persistent_kernel<2>
                        : (p.stage ? (const void*)ppo_persistent_kernel<1> : (const void*)ppo_persistent_kernel<0>);
  PRB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, kPpoThreads, smem));
  if (occ < 1) return 0;
  const int work = std::max(2 * ((p.mb + p.R - 1) / p.R), ws.ntiles * ws.RS);
  return std::min(work, a->ctx->num_sms * occ);
}

void launch_persistent(const PpoArgs& p, prb_agent a, PpoWorkspace& ws, double ent, int64_t steps, int grid,
                       cudaStream_t s) {
  PpoArgs pa = p;
  pa.trace = nullptr;
  GradArgs g = make_grad_args(p, a, ws, ent, 1);
  g.trace = nullptr;
  ws.bar.ensure(4);  // [0] barrier arrivals, [1] unused, [2..3] per-step non-finite flags
  PRB_CUDA(cudaMemsetAsync(ws.bar.p, 0, ws.bar.bytes(), s));
  unsigned int* bar = reinterpret_cast<unsigned int*>(ws.bar.p);
  int32_t* flags = ws.bar.p + 2;
  unsigned long long* trace = nullptr;
  if (debug_env("PRB_PPO_TRACE")) {  // [grid][10] phase stamps, then fwd_delta_block's 2 x 16 clock64 marks
    ws.ptrace.alloc((size_t)grid * 16 + 32);
    PRB_CUDA(cudaMemsetAsync(ws.ptrace.p, 0, ws.ptrace.bytes(), s));
    trace = ws.ptrace.p;
    pa.trace = ws.ptrace.p + (size_t)grid * 16;
  }
  ws.bias.ensure((size_t)steps);
  float2* bias_tab = ws.bias.p;
  pa.nospec = debug_env("PRB_PPO_NOSPEC") ? 1 : 0;
  if (p.r8 && p.stage && !debug_env("PRB_PPO_CPASYNC")) {  // PRB_PPO_CPASYNC=1: per-thread cp.async staging (A/B)
    pa.img_c = (int)staged_floats(p.actor, 1);
    const size_t nimg = (size_t)pa.img_c + staged_floats(p.critic, 1);
    ws.wimg.ensure(nimg);
    PRB_CUDA(cudaMemsetAsync(ws.wimg.p, 0, nimg * sizeof(float), s));  // row padding
    pa.wimg = ws.wimg.p;
  }
  if (p.r8 && !debug_env("PRB_PPO_NOTAB")) {  // PRB_PPO_NOTAB=1: rows resolved inline (A/B)
    ws.rtab.ensure(2 * (size_t)p.mb);
    pa.rtab = ws.rtab.p;
  }
  void* args[] = {&pa, &g, &steps, &bar, &flags, &bias_tab, &trace};
  const size_t smem = persistent_smem(p);
  launch_coop(p.r8 ? (const void*)ppo_persistent_kernel<2>
                   : (p.stage ? (const void*)ppo_persistent_kernel<1> : (const void*)ppo_persistent_kernel<0>),
              grid, smem, s, args);
}

// The tensor-core update (ppo_tc.cu) covers the stock-pod nets: actor S-64-64-A, critic
// S-64-64-1 with A <= 32, minibatches of <= 1,024 rows (<= 8 CTAs of 128 rows per learner), and
// inputs that fit its 192-column X tile (<= 32 private features + <= 156 others + the ones column).
bool ppo_tc_supported(prb_agent a, prb_rollout r, int mb, int mode) {
  if (mode != 1) return false;
  const std::vector<size_t> ad = {a->S, 64, 64, a->A}, cd = {a->S, 64, 64, 1};
  if (a->adims != ad || a->cdims != cd || a->A > 32 || mb > kPpoTcMaxRows || mb < 1) return false;
  const size_t nrest = r->obs_mode == 1 ? 5 * (size_t)r->K : a->S - std::min<size_t>(a->S, 32);
  const size_t npriv = r->obs_mode == 1 ? r->Sp : std::min<size_t>(a->S, 32);
  return npriv <= 32 && nrest <= 156;  // X and the fp32 gather staging fit (ppo_tc.cu)
}

// The launch-wide part of the tensor-core update (net layout, buffer shape, schedule); the image
// position table lives in `ws` (computed once per workspace and shape).
PpoTcArgs make_tc_shape(const PpoArgs& p, prb_agent a, prb_rollout r, PpoWorkspace& ws, int64_t steps,
                        cudaStream_t s) {
  PpoTcArgs t{};
  t.S = p.S;
  t.A = p.A;
  t.P = p.P;
  t.Pp = (int)((a->P + 2 + 31) & ~size_t(31));
  for (int l = 0; l < 3; ++l) {
    t.a_w[l] = (int)a->aoff[l];
    t.c_w[l] = (int)a->coff[l];
  }
  t.log_std = (int)a->Pa;
  t.obs_mode = r->obs_mode;
  t.Sp = (int)r->Sp;
  t.F = 5 * r->K;
  t.npriv = r->obs_mode == 1 ? (int)r->Sp : std::min(p.S, 32);
  t.nrest = r->obs_mode == 1 ? t.F : p.S - t.npriv;
  t.ones_col = 32 + t.nrest;
  t.N = p.N;
  t.n = p.n;
  t.nmb = p.nmb;
  t.bits = p.bits;
  t.mb = p.mb;
  t.C = (p.mb + 127) / 128;
  t.steps = steps;
  t.clip = (float)p.clip;
  t.ent = (float)p.ent;
  t.vf = (float)p.vf;
  t.b1 = a->beta1;
  t.b2 = a->beta2;
  t.eps = (float)a->eps;
  const std::vector<int> key = {t.S, t.A, t.P, t.npriv, t.nrest, t.a_w[0], t.c_w[0]};
  if (ws.tc_pos_key != key) {
    ws.tc_pos.ensure((size_t)t.P);
    ppo_tc_image_positions(t, ws.tc_pos.p, s);
    ws.tc_pos_key = key;
  }
  t.imgpos = ws.tc_pos.p;
  return t;
}

// One learner of a tensor-core launch: its agent (dst, trained in place), its workspace and buffer.
PpoTcChain make_tc_chain(const PpoTcArgs& t, prb_agent dst, prb_rollout r, PpoWorkspace& ws, const uint32_t* perm,
                         uint64_t seed, cudaStream_t s) {
  ws.tc_img.ensure(kPpoTcImgBytes);
  ws.tc_slab.ensure((size_t)t.C * t.Pp);
  ws.tc_stats.ensure(4);
  PRB_CUDA(cudaMemsetAsync(ws.tc_img.p, 0, kPpoTcImgBytes, s));  // padding of the operand blocks
  PRB_CUDA(cudaMemsetAsync(ws.tc_stats.p, 0, 4 * sizeof(double), s));
  ws.tc_sync.ensure(16);
  PRB_CUDA(cudaMemsetAsync(ws.tc_sync.p, 0, 16 * sizeof(uint32_t), s));
  PpoTcChain c{};
  c.sync = ws.tc_sync.p;
  c.params = dst->d_params.p;
  c.m = dst->d_m.p;
  c.v = dst->d_v.p;
  c.t = dst->d_t.p;
  c.grads = dst->d_grads.p;
  c.img = ws.tc_img.p;
  c.slab = ws.tc_slab.p;
  c.stats = ws.tc_stats.p;
  c.status = dst->d_status.p;
  c.perm = perm;
  c.seed = seed;
  c.lr = (float)dst->lr;
  c.obs = r->d_obs.p;
  c.row = r->d_row.p;
  c.feat = r->d_feat;
  c.act = r->d_act.p;
  c.logp = r->d_logp.p;
  c.adv = r->d_adv.p;
  c.ret = r->d_ret.p;
  c.advstat = r->d_advstat.p;
  return c;
}

// Uploads the chain descriptors into `buf` and points t at them (synchronous: the host vector
// may die on return).
void upload_chains(PpoTcArgs& t, const std::vector<PpoTcChain>& chains, DevBuf<PpoTcChain>& buf, cudaStream_t s) {
  buf.ensure(chains.size());
  PRB_CUDA(cudaMemcpyAsync(buf.p, chains.data(), chains.size() * sizeof(PpoTcChain), cudaMemcpyHostToDevice, s));
  PRB_CUDA(cudaStreamSynchronize(s));
  t.chains = buf.p;
}

std::string status_message(int detail) {
  switch (detail) {
    case 10: return "ppo_losses: policy_loss is non-finite";
    case 11: return "ppo_losses: value_loss is non-finite";
    case 12: return "ppo_losses: entropy is non-finite";
    default: return "adam_step: non-finite gradient, step aborted";
  }
}

void check_status(prb_agent a) {
  int32_t st[2];
  PRB_CUDA(cudaMemcpyAsync(st, a->d_status.p, 2 * sizeof(int32_t), cudaMemcpyDeviceToHost, a->ctx->stream));
  a->ctx->sync();
  if (st[0] != 0) {
    PRB_CUDA(cudaMemsetAsync(a->d_status.p, 0, 4 * sizeof(int32_t), a->ctx->stream));
    a->ctx->sync();
    fail(st[0], status_message(st[1]));
  }
}

void set_smem_attr() {  // per device (ensure_smem_attr); the caller's DeviceScope made it current
  const void* fns[] = {(const void*)ppo_fwd_delta_kernel<0>, (const void*)ppo_fwd_delta_kernel<1>,
                       (const void*)ppo_fwd_delta_kernel<2>, (const void*)ppo_persistent_kernel<0>,
                       (const void*)ppo_persistent_kernel<1>, (const void*)ppo_persistent_kernel<2>};
  for (const void* f : fns) ensure_smem_attr(f, kSmemBudget);
  ensure_smem_attr((const void*)ppo_grad_kernel, 2 * kGChunk * kGLd * sizeof(float));
}

std::vector<uint32_t> ref_rows_to_device(prb_rollout r, const uint64_t* rows, size_t count) {
  std::vector<uint32_t> out(count);
  const size_t n = r->N * r->H;
  for (size_t i = 0; i < count; ++i) {
    PRB_REQUIRE(rows[i] < n, PRB_ERR_USAGE, "ppo: permutation index out of range");
    const size_t e = rows[i] / r->H, h = rows[i] % r->H;  // reference env-major -> device time-major
    out[i] = (uint32_t)(h * r->N + e);
  }
  return out;
}

}  // namespace

void prb_gae_launch(prb_ctx ctx, const float* rew, const float* val, const uint8_t* done, const float* boot, size_t N,
                    size_t H, double gamma, double lambda, float* adv, float* ret, double* stat, int normalize);

extern "C" {

int prb_ppo_update(prb_agent src, prb_rollout r, const prb_ppo_config* cfg, uint64_t seed, const uint64_t* perm,
                   prb_agent dst, prb_ppo_stats* stats) {
  return guard([&] {
    DeviceScope dev_(src ? src->ctx : nullptr);
    PRB_REQUIRE(src && r && cfg && dst, PRB_ERR_USAGE, "ppo_update: NULL argument");
    // PpoConfig::validate ppo.hpp:29-37
    PRB_REQUIRE(cfg->gamma > 0.0 && cfg->gamma <= 1.0, PRB_ERR_CONFIG, "ppo.gamma must be in (0, 1]");
    PRB_REQUIRE(cfg->gae_lambda >= 0.0 && cfg->gae_lambda <= 1.0, PRB_ERR_CONFIG, "ppo.gae_lambda must be in [0, 1]");
    PRB_REQUIRE(cfg->clip_eps > 0.0, PRB_ERR_CONFIG, "ppo.clip_eps must be > 0");
    PRB_REQUIRE(cfg->minibatch_size <= cfg->buffer_size, PRB_ERR_CONFIG, "ppo.minibatch_size exceeds ppo.buffer_size");
    PRB_REQUIRE(cfg->minibatch_size > 0, PRB_ERR_CONFIG, "ppo.minibatch_size must be > 0");
    const size_t n = r->N * r->H;
    PRB_REQUIRE(r->full, PRB_ERR_USAGE, "ppo_update: buffer has 0 of " + std::to_string(n) + " transitions");
    PRB_REQUIRE(n >= cfg->minibatch_size, PRB_ERR_USAGE,
                "ppo_update: buffer length " + std::to_string(n) + " shorter than minibatch_size " +
                    std::to_string(cfg->minibatch_size));
    PRB_REQUIRE(src->adims == dst->adims && src->cdims == dst->cdims && src->S == r->S && src->A == r->A,
                PRB_ERR_USAGE, "ppo_update: agent/buffer shapes disagree");
    PRB_REQUIRE(cfg->minibatch_size < (1u << 30), PRB_ERR_CONFIG, "ppo.minibatch_size too large");
    set_smem_attr();
    cudaStream_t s = dst->ctx->stream;
    // ppo_update is pure w.r.t. its inputs (ppo.hpp:246-248): with src == dst the agent is
    // snapshotted first and restored if the update fails, so a NumericError leaves it intact
    DevBuf<float> snap;
    int64_t snap_t = 0;
    const double snap_lr = dst->lr;
    if (src != dst) {
      int rc = prb_agent_copy(dst, src);
      if (rc) fail(rc, prb_last_error());
    } else {
      snap.alloc(3 * dst->P);
      PRB_CUDA(cudaMemcpyAsync(snap.p, dst->d_params.p, dst->P * sizeof(float), cudaMemcpyDeviceToDevice, s));
      PRB_CUDA(cudaMemcpyAsync(snap.p + dst->P, dst->d_m.p, dst->P * sizeof(float), cudaMemcpyDeviceToDevice, s));
      PRB_CUDA(cudaMemcpyAsync(snap.p + 2 * dst->P, dst->d_v.p, dst->P * sizeof(float), cudaMemcpyDeviceToDevice, s));
      PRB_CUDA(cudaMemcpyAsync(&snap_t, dst->d_t.p, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
      dst->ctx->sync();
    }
    try {
    dst->lr = cfg->learning_rate;  // ppo.hpp:265
    PRB_CUDA(cudaMemsetAsync(dst->d_status.p, 0, 4 * sizeof(int32_t), s));
    prb_gae_launch(r->ctx, r->d_rew.p, r->d_val.p, r->d_done.p, r->d_boot.p, r->N, r->H, cfg->gamma, cfg->gae_lambda,
                   r->d_adv.p, r->d_ret.p, r->d_advstat.p, 1);
    if (r->ctx->stream != s) r->ctx->sync();
    r->gae_valid = true;
    r->normalized = true;
    if (!dst->ppo_ws)  // device workspace kept with the agent: no cudaMalloc/cudaFree per update
      dst->ppo_ws = std::shared_ptr<void>(new PpoWorkspace, [](void* w) { delete static_cast<PpoWorkspace*>(w); });
    PpoWorkspace& ws = *static_cast<PpoWorkspace*>(dst->ppo_ws.get());
    const int mb = (int)cfg->minibatch_size;
    PpoArgs p = make_args(dst, r, cfg, seed, ws, mb);
    const size_t steps = (size_t)cfg->epochs_per_update * p.nmb;
    if (perm) {
      std::vector<uint32_t> dev = ref_rows_to_device(r, perm, (size_t)cfg->epochs_per_update * n);
      ws.perm.ensure(dev.size());
      PRB_CUDA(cudaMemcpyAsync(ws.perm.p, dev.data(), dev.size() * sizeof(uint32_t), cudaMemcpyHostToDevice, s));
      p.perm = ws.perm.p;
      dst->ctx->sync();
    }
    PRB_CUDA(cudaMemsetAsync(ws.step.p, 0, sizeof(int64_t), s));
    PRB_CUDA(cudaMemsetAsync(ws.stats.p, 0, 4 * sizeof(double), s));
    // Minibatch steps are identical launches (the counter is on device):
    // capture a block of them once as a CUDA graph and replay it.
    const size_t kGraphSteps = 32;
    const int pgrid = persistent_grid(p, dst, ws);
    if (steps > 0 && ppo_tc_supported(dst, r, mb, src->ppo_mode)) {  // one learner's CTAs run the whole chain
      PpoTcArgs ta = make_tc_shape(p, dst, r, ws, (int64_t)steps, s);
      upload_chains(ta, {make_tc_chain(ta, dst, r, ws, p.perm, p.seed, s)}, ws.tc_chain, s);
      const char* tpath = debug_env("PRB_PPO_TC_TRACE");  // debug: phase marks of one step
      DevBuf<unsigned long long> tbuf;
      if (tpath) {
        tbuf.alloc(32);
        PRB_CUDA(cudaMemsetAsync(tbuf.p, 0, tbuf.bytes(), s));
        ta.trace = tbuf.p;
      }
      {
        ProfScope prof(dst->ctx, kProfPpoFwdBwd);
        launch_ppo_tc(ta, 1, s);
      }
      PRB_CHECK_LAUNCH();
      PRB_CUDA(cudaStreamSynchronize(s));
      if (tpath) {
        unsigned long long h[32];
        PRB_CUDA(cudaMemcpy(h, tbuf.p, sizeof(h), cudaMemcpyDeviceToHost));
        if (FILE* f = fopen(tpath, "w")) {
          for (int i = 0; i < 32; ++i) fprintf(f, "%d %lld\n", i, h[i] ? (long long)(h[i] - h[0]) : -1LL);
          fclose(f);
        }
      }
      PRB_CUDA(cudaMemcpyAsync(ws.stats.p, ws.tc_stats.p, 4 * sizeof(double), cudaMemcpyDeviceToDevice, s));
    } else if (pgrid > 0 && steps > 0) {
      {
        ProfScope prof(dst->ctx, kProfPpoFwdBwd);
        launch_persistent(p, dst, ws, cfg->entropy_coef, (int64_t)steps, pgrid, s);
      }
      PRB_CUDA(cudaStreamSynchronize(s));
    } else if (steps >= kGraphSteps) {
      cudaGraph_t graph;
      cudaGraphExec_t exec;
      PRB_CUDA(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
      for (size_t i = 0; i < kGraphSteps; ++i) launch_step(p, dst, ws, cfg->entropy_coef, 1, s);
      PRB_CUDA(cudaStreamEndCapture(s, &graph));
      PRB_CUDA(cudaGraphInstantiate(&exec, graph, 0));
      for (size_t i = 0; i + kGraphSteps <= steps; i += kGraphSteps) PRB_CUDA(cudaGraphLaunch(exec, s));
      for (size_t i = (steps / kGraphSteps) * kGraphSteps; i < steps; ++i) launch_step(p, dst, ws, cfg->entropy_coef, 1, s);
      PRB_CUDA(cudaStreamSynchronize(s));
      cudaGraphExecDestroy(exec);
      cudaGraphDestroy(graph);
    } else {
      for (size_t i = 0; i < steps; ++i) launch_step(p, dst, ws, cfg->entropy_coef, 1, s);
    }
    PRB_CHECK_LAUNCH();
    if (const char* tp = debug_env("PRB_PPO_TRACE")) {  // debug: globaltimer marks of the last step's ppo_grad CTAs
      DevBuf<unsigned long long>& tb = ws.ptrace.p ? ws.ptrace : ws.trace;  // persistent: [grid][10] stamps
      std::vector<unsigned long long> h(tb.n);
      PRB_CUDA(cudaMemcpy(h.data(), tb.p, tb.bytes(), cudaMemcpyDeviceToHost));
      if (FILE* f = fopen(tp, "wb")) {
        fwrite(h.data(), 8, h.size(), f);
        fclose(f);
      }
    }
    check_status(dst);
    double st[4];
    PRB_CUDA(cudaMemcpyAsync(st, ws.stats.p, sizeof(st), cudaMemcpyDeviceToHost, s));
    dst->ctx->sync();
    if (stats) {
      stats->minibatches = (uint64_t)st[3];
      const double inv = st[3] > 0 ? 1.0 / st[3] : 0.0;
      stats->mean_policy_loss = st[0] * inv;
      stats->mean_value_loss = st[1] * inv;
      stats->mean_entropy = st[2] * inv;
    }
    } catch (...) {
      if (snap.p) {  // src == dst: put the input back
        cudaStreamSynchronize(s);
        cudaMemcpyAsync(dst->d_params.p, snap.p, dst->P * sizeof(float), cudaMemcpyDeviceToDevice, s);
        cudaMemcpyAsync(dst->d_m.p, snap.p + dst->P, dst->P * sizeof(float), cudaMemcpyDeviceToDevice, s);
        cudaMemcpyAsync(dst->d_v.p, snap.p + 2 * dst->P, dst->P * sizeof(float), cudaMemcpyDeviceToDevice, s);
        cudaMemcpyAsync(dst->d_t.p, &snap_t, sizeof(int64_t), cudaMemcpyHostToDevice, s);
        cudaStreamSynchronize(s);
        dst->lr = snap_lr;
      }
      throw;
    }
  });
}

int prb_ppo_update_learners(const prb_agent* srcs, const prb_rollout* rollouts, size_t L, const prb_ppo_config* cfg,
                            const uint64_t* seeds, const prb_agent* dsts, prb_ppo_stats* stats) {
  return guard([&] {
    PRB_REQUIRE(srcs && rollouts && cfg && seeds && dsts && L > 0, PRB_ERR_USAGE, "ppo_update_learners: NULL argument");
    DeviceScope dev_(dsts[0] ? dsts[0]->ctx : nullptr);
    PRB_REQUIRE(cfg->gamma > 0.0 && cfg->gamma <= 1.0, PRB_ERR_CONFIG, "ppo.gamma must be in (0, 1]");
    PRB_REQUIRE(cfg->gae_lambda >= 0.0 && cfg->gae_lambda <= 1.0, PRB_ERR_CONFIG, "ppo.gae_lambda must be in [0, 1]");
    PRB_REQUIRE(cfg->clip_eps > 0.0, PRB_ERR_CONFIG, "ppo.clip_eps must be > 0");
    PRB_REQUIRE(cfg->minibatch_size > 0 && cfg->minibatch_size <= cfg->buffer_size, PRB_ERR_CONFIG,
                "ppo.minibatch_size must be in [1, buffer_size]");
    const prb_rollout r0 = rollouts[0];
    PRB_REQUIRE(r0, PRB_ERR_USAGE, "ppo_update_learners: NULL rollout");
    const size_t n = r0->N * r0->H;
    for (size_t l = 0; l < L; ++l) {
      const prb_agent src = srcs[l], dst = dsts[l];
      const prb_rollout r = rollouts[l];
      PRB_REQUIRE(src && dst && r && src != dst, PRB_ERR_USAGE, "ppo_update_learners: NULL or aliased agent");
      PRB_REQUIRE(r->full, PRB_ERR_USAGE, "ppo_update: buffer has 0 of " + std::to_string(r->N * r->H) + " transitions");
      PRB_REQUIRE(r->N == r0->N && r->H == r0->H && r->S == r0->S && r->A == r0->A && r->obs_mode == r0->obs_mode &&
                      r->K == r0->K,
                  PRB_ERR_USAGE, "ppo_update_learners: rollout buffers of different shapes");
      PRB_REQUIRE(src->adims == dst->adims && src->cdims == dst->cdims && src->S == r->S && src->A == r->A &&
                      dst->ctx->device == dsts[0]->ctx->device,
                  PRB_ERR_USAGE, "ppo_update_learners: agent/buffer shapes or devices disagree");
      for (size_t k = 0; k < l; ++k)
        PRB_REQUIRE(dsts[k] != dst, PRB_ERR_USAGE, "ppo_update_learners: a destination agent appears twice");
    }
    PRB_REQUIRE(n >= cfg->minibatch_size, PRB_ERR_USAGE,
                "ppo_update: buffer length " + std::to_string(n) + " shorter than minibatch_size " +
                    std::to_string(cfg->minibatch_size));
    const int mb = (int)cfg->minibatch_size;
    if (!ppo_tc_supported(dsts[0], r0, mb, 1)) {
      // other shapes (e.g. PointMass 3x256): each learner's own update on the whole-GPU SIMT path,
      // one after another; a learner whose gate fails keeps its last accepted step and the
      // others still run (the first failure is reported)
      int first = 0;
      std::string msg;
      for (size_t l = 0; l < L; ++l) {
        const int rc = prb_ppo_update(srcs[l], rollouts[l], cfg, seeds[l], nullptr, dsts[l], stats ? &stats[l] : nullptr);
        if (rc && !first) {
          first = rc;
          msg = prb_last_error();
        }
      }
      if (first) fail(first, msg);
      return;
    }
    cudaStream_t s = dsts[0]->ctx->stream;
    // GAE + normalisation once per distinct buffer (learners of one pod share it)
    for (size_t l = 0; l < L; ++l) {
      bool seen = false;
      for (size_t k = 0; k < l; ++k) seen |= rollouts[k] == rollouts[l];
      if (seen) continue;
      prb_rollout r = rollouts[l];
      prb_gae_launch(r->ctx, r->d_rew.p, r->d_val.p, r->d_done.p, r->d_boot.p, r->N, r->H, cfg->gamma,
                     cfg->gae_lambda, r->d_adv.p, r->d_ret.p, r->d_advstat.p, 1);
      if (r->ctx->stream != s) r->ctx->sync();
      r->gae_valid = true;
      r->normalized = true;
    }
    for (size_t l = 0; l < L; ++l) {
      int rc = prb_agent_copy(dsts[l], srcs[l]);
      if (rc) fail(rc, prb_last_error());
      dsts[l]->lr = cfg->learning_rate;  // ppo.hpp:265
      PRB_CUDA(cudaMemsetAsync(dsts[l]->d_status.p, 0, 4 * sizeof(int32_t), s));
      if (!dsts[l]->ppo_ws)
        dsts[l]->ppo_ws = std::shared_ptr<void>(new PpoWorkspace, [](void* w) { delete static_cast<PpoWorkspace*>(w); });
    }
    PpoWorkspace& ws0 = *static_cast<PpoWorkspace*>(dsts[0]->ppo_ws.get());
    PpoArgs p = make_args(dsts[0], r0, cfg, seeds[0], ws0, mb);
    const int64_t steps = (int64_t)cfg->epochs_per_update * p.nmb;
    if (steps == 0) return;
    PpoTcArgs t = make_tc_shape(p, dsts[0], r0, ws0, steps, s);
    std::vector<PpoTcChain> chains;
    for (size_t l = 0; l < L; ++l) {
      PpoWorkspace& ws = *static_cast<PpoWorkspace*>(dsts[l]->ppo_ws.get());
      chains.push_back(make_tc_chain(t, dsts[l], rollouts[l], ws, nullptr, seeds[l], s));
    }
    DevBuf<PpoTcChain> cbuf;
    upload_chains(t, chains, cbuf, s);
    const char* tpath = debug_env("PRB_PPO_TC_TRACE");  // debug: phase marks of chain 0, step 8
    DevBuf<unsigned long long> tbuf;
    if (tpath) {
      tbuf.alloc(32);
      PRB_CUDA(cudaMemsetAsync(tbuf.p, 0, tbuf.bytes(), s));
      t.trace = tbuf.p;
    }
    {
      ProfScope prof(dsts[0]->ctx, kProfPpoFwdBwd);
      launch_ppo_tc(t, (int)L, s);
    }
    PRB_CHECK_LAUNCH();
    PRB_CUDA(cudaStreamSynchronize(s));
    if (tpath) {
      unsigned long long h[32];
      PRB_CUDA(cudaMemcpy(h, tbuf.p, sizeof(h), cudaMemcpyDeviceToHost));
      if (FILE* f = fopen(tpath, "w")) {
        for (int i = 0; i < 32; ++i) fprintf(f, "%d %lld\n", i, h[i] ? (long long)(h[i] - h[0]) : -1LL);
        fclose(f);
      }
    }
    // every learner's status and statistics in one batch of copies, one synchronisation
    struct Rec {
      double h[4];
      int32_t st[2];
      int32_t pad[2];
    };
    Rec* rec = static_cast<Rec*>(dsts[0]->ctx->pinned_staging(L * sizeof(Rec)));
    for (size_t l = 0; l < L; ++l) {
      PpoWorkspace& ws = *static_cast<PpoWorkspace*>(dsts[l]->ppo_ws.get());
      PRB_CUDA(cudaMemcpyAsync(rec[l].st, dsts[l]->d_status.p, 2 * sizeof(int32_t), cudaMemcpyDeviceToHost, s));
      if (stats) PRB_CUDA(cudaMemcpyAsync(rec[l].h, ws.tc_stats.p, 4 * sizeof(double), cudaMemcpyDeviceToHost, s));
    }
    PRB_CUDA(cudaStreamSynchronize(s));
    int first_code = 0, first_detail = 0;
    for (size_t l = 0; l < L; ++l) {
      const int32_t* st = rec[l].st;
      if (st[0] && !first_code) {
        first_code = st[0];
        first_detail = st[1];
      }
      if (st[0]) PRB_CUDA(cudaMemsetAsync(dsts[l]->d_status.p, 0, 4 * sizeof(int32_t), s));
      if (stats) {
        const double* h = rec[l].h;
        stats[l].minibatches = (uint64_t)h[3];
        const double inv = h[3] > 0 ? 1.0 / h[3] : 0.0;
        stats[l].mean_policy_loss = h[0] * inv;
        stats[l].mean_value_loss = h[1] * inv;
        stats[l].mean_entropy = h[2] * inv;
      }
    }
    PRB_CUDA(cudaStreamSynchronize(s));
    if (first_code) fail(first_code, status_message(first_detail));
  });
}

int prb_ppo_loss_grads(prb_agent a, prb_rollout r, const uint64_t* rows, size_t n, const prb_ppo_config* cfg,
                       double* grads, double* losses) {
  return guard([&] {
    DeviceScope dev_(a ? a->ctx : nullptr);
    PRB_REQUIRE(a && r && rows && cfg, PRB_ERR_USAGE, "ppo_loss_grads: NULL argument");
    PRB_REQUIRE(r->gae_valid, PRB_ERR_USAGE, "ppo_loss_grads: call prb_gae first");
    PRB_REQUIRE(n > 0 && n < (1u << 30), PRB_ERR_DIMENSION, "ppo_loss_grads: bad minibatch size");
    set_smem_attr();
    cudaStream_t s = a->ctx->stream;
    PpoWorkspace ws;
    PpoArgs p = make_args(a, r, cfg, 0, ws, (int)n);
    std::vector<uint32_t> dev = ref_rows_to_device(r, rows, n);
    ws.perm.alloc(n);
    PRB_CUDA(cudaMemcpyAsync(ws.perm.p, dev.data(), n * sizeof(uint32_t), cudaMemcpyHostToDevice, s));
    p.perm = ws.perm.p;
    p.n = (uint32_t)n;  // one "epoch" whose permutation is exactly `rows`
    p.nmb = 1;
    PRB_CUDA(cudaMemsetAsync(ws.step.p, 0, sizeof(int64_t), s));
    PRB_CUDA(cudaMemsetAsync(ws.stats.p, 0, 4 * sizeof(double), s));
    PRB_CUDA(cudaMemsetAsync(a->d_status.p, 0, 4 * sizeof(int32_t), s));
    launch_step(p, a, ws, cfg->entropy_coef, 0, s);
    PRB_CHECK_LAUNCH();
    a->ctx->sync();
    int32_t st[2];
    PRB_CUDA(cudaMemcpy(st, a->d_status.p, sizeof(st), cudaMemcpyDeviceToHost));
    double sums[4];
    PRB_CUDA(cudaMemcpy(sums, ws.stats.p, sizeof(sums), cudaMemcpyDeviceToHost));
    if (losses) {
      losses[0] = sums[0];
      losses[1] = sums[1];
      losses[2] = sums[2];
    }
    if (st[0] != 0) {
      PRB_CUDA(cudaMemsetAsync(a->d_status.p, 0, 4 * sizeof(int32_t), a->ctx->stream));
      a->ctx->sync();
      fail(st[0], status_message(st[1]));
    }
    if (grads) {
      std::vector<float> g(a->P);
      PRB_CUDA(cudaMemcpy(g.data(), a->d_grads.p, a->P * sizeof(float), cudaMemcpyDeviceToHost));
      for (size_t i = 0; i < a->P; ++i) grads[i] = g[i];
    }
  });
}

}  // extern "C"
