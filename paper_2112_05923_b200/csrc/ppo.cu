// ppo.cu -- PPO update on device (ppo_update ppo.hpp:249-296,
// detail::ppo_loss_grads ppo.hpp:116-188, mlp_backward_accumulate
// nn.hpp:105-132, adam_step nn.hpp:164-182).
//
// One minibatch step = three stream-ordered kernels, all parameters and the
// whole rollout staying in HBM/L2:
//   1. ppo_fwd_bwd: each CTA gathers R rows of the minibatch (permutation
//      computed on the fly: a keyed Feistel bijection of the buffer, or the
//      injected reference permutation), rebuilds the observation (compact stock
//      rows + shared feature row), stages the whole actor+critic weight set in
//      shared memory (row stride out+1: conflict-free for the forward's
//      column walk and the backward's row walk), runs the forward with cached
//      activations, forms the clipped-surrogate / value / entropy head
//      gradients (subgradient ties as ppo.hpp:146), backpropagates, and writes
//      its partial dW/db/dlog_std and loss sums to a [CTA][P] slab.
//   2. ppo_reduce: deterministic fixed-order sum of the partials, entropy term,
//      finiteness gate (losses first, then gradients -- reference order), and
//      the last CTA advances t / the minibatch counter.
//   3. adam (agent.cu), skipped by the gate so a non-finite step leaves the
//      state untouched (nn.hpp:169-171).
// The minibatch counter lives on device, so a run of steps is one CUDA graph.
#include <algorithm>
#include <cmath>
#include <cstring>

#include "mlp_simt.cuh"
#include "policy_internal.h"
#include "prb_internal.h"
#include "rng.cuh"

using namespace prb;

namespace {

constexpr float kLogTwoPiF = 1.8378770664093454836f;
constexpr int kPpoThreads = 256;
constexpr size_t kSmemBudget = 220 * 1024;

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
  const int64_t* step;  // device minibatch counter (epoch = step / nmb)
  double clip, ent, vf;
  float* partial;  // [grid][Pext]
  int32_t* status;
  int ldw;  // max hidden width rounded to 4
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

// floats of the staged weight set: every layer of both nets at row stride out+1
__host__ __device__ inline size_t staged_floats(const PpoArgs& a) {
  size_t n = 0;
  for (int l = 0; l < a.actor.nl; ++l) n += (size_t)a.actor.dims[l] * (a.actor.dims[l + 1] + 1);
  for (int l = 0; l < a.critic.nl; ++l) n += (size_t)a.critic.dims[l] * (a.critic.dims[l + 1] + 1);
  return (n + 3) & ~size_t(3);
}

struct Smem {
  float* w;  // staged weights (nullptr when not staged)
  float* x;
  float* aa[kMaxLayers];
  int lda[kMaxLayers];
  float* ca[kMaxLayers];
  int ldc[kMaxLayers];
  float* d0;
  float* d1;
  float* actn;
  float* misc;  // [R8][4]: old_lp, adv_norm, ret, -
  float* tmp;   // [R8][ldA]
  float* loss;  // [R8][2]
};

__host__ __device__ inline size_t carve(const PpoArgs& a, float* base, Smem* s) {
  const int R8 = (a.R + 7) & ~7;
  const int ldx = (a.S + 3) & ~3;
  const int ldA = (a.A + 3) & ~3;
  size_t o = 0;
  auto take = [&](size_t n) {
    float* p = base ? base + o : nullptr;
    o += (n + 3) & ~size_t(3);
    return p;
  };
  float* w = a.stage ? take(staged_floats(a)) : nullptr;
  if (s) s->w = w;
  float* x = take((size_t)R8 * ldx);
  if (s) s->x = x;
  for (int l = 0; l < a.actor.nl; ++l) {
    const int ld = (a.actor.dims[l + 1] + 3) & ~3;
    float* p = take((size_t)R8 * ld);
    if (s) {
      s->aa[l] = p;
      s->lda[l] = ld;
    }
  }
  for (int l = 0; l < a.critic.nl; ++l) {
    const int ld = (a.critic.dims[l + 1] + 3) & ~3;
    float* p = take((size_t)R8 * ld);
    if (s) {
      s->ca[l] = p;
      s->ldc[l] = ld;
    }
  }
  const int ldd = a.ldw > ldA ? a.ldw : ldA;
  float* d0 = take((size_t)R8 * ldd);
  float* d1 = take((size_t)R8 * ldd);
  float* actn = take((size_t)R8 * ldA);
  float* misc = take((size_t)R8 * 4);
  float* tmp = take((size_t)R8 * ldA);
  float* loss = take((size_t)R8 * 2);
  if (s) {
    s->d0 = d0;
    s->d1 = d1;
    s->actn = actn;
    s->misc = misc;
    s->tmp = tmp;
    s->loss = loss;
  }
  return o * sizeof(float);
}

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

// gW[k][j] = sum_r in[r][k] d[r][j]; gb[j] = sum_r d[r][j]   (matmul_tn + column_sums, tensor.hpp:85-183)
__device__ __forceinline__ void grad_w_tile(const float* s_in, int ldi, int in, const float* s_d, int ldd, int out,
                                            int nrows, float* __restrict__ gW) {
  const int TJ = out > 32 ? 64 : 32;
  const int KT = blockDim.x / TJ;
  const int jt = threadIdx.x % TJ, kt = threadIdx.x / TJ;
  for (int j = jt; j < out; j += TJ) {
    for (int k = kt; k < in; k += KT) {
      float acc = 0.0f;
      for (int r = 0; r < nrows; ++r) acc = fmaf(s_in[r * ldi + k], s_d[r * ldd + j], acc);
      gW[(size_t)k * out + j] = acc;
    }
    if (kt == 0) {
      float acc = 0.0f;
      for (int r = 0; r < nrows; ++r) acc += s_d[r * ldd + j];
      gW[(size_t)in * out + j] = acc;
    }
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

__global__ void __launch_bounds__(kPpoThreads) ppo_fwd_bwd_kernel(PpoArgs a) {
  if (a.status[0] != 0) return;
  extern __shared__ __align__(16) float smem[];
  Smem s;
  carve(a, smem, &s);
  const int64_t step = *a.step;
  const int R = a.R;
  const int ldx = (a.S + 3) & ~3;
  const int A = a.A, ldA = (A + 3) & ~3;
  const int q0 = blockIdx.x * R;
  const int nrows = min(R, a.mb - q0);
  const double mean = a.advstat[0], denom = a.advstat[1];
  float* wa = nullptr;
  float* wc = nullptr;
  if (a.stage) {
    wa = s.w;
    size_t na = 0;
    for (int l = 0; l < a.actor.nl; ++l) na += (size_t)a.actor.dims[l] * (a.actor.dims[l + 1] + 1);
    wc = s.w + na;
    stage_weights(a, a.actor, wa);
    stage_weights(a, a.critic, wc);
  }
  // the gather below overlaps with the weight copies in flight; waited before the forward
  const LayerPtrs lpa = layer_ptrs(a, a.actor, wa), lpc = layer_ptrs(a, a.critic, wc);
  // ---- gather (gather_minibatch ppo.hpp:83-103) ----
  for (int r = threadIdx.x / 32; r < nrows; r += blockDim.x / 32) {
    const uint32_t i = mb_row(a, step, (uint32_t)(q0 + r));
    const int lane = threadIdx.x & 31;
    if (a.obs_mode == 1) {
      const uint32_t h = i / a.N;
      const float* fr = a.feat + (size_t)a.row[h] * (a.S - a.Sp);
      for (int c = lane; c < a.S; c += 32)
        s.x[r * ldx + c] = (c < a.Sp) ? a.obs[(size_t)i * a.Sp + c] : fr[c - a.Sp];
    } else {
      for (int c = lane; c < a.S; c += 32) s.x[r * ldx + c] = a.obs[(size_t)i * a.S + c];
    }
    for (int c = lane; c < A; c += 32) s.actn[r * ldA + c] = a.act[(size_t)i * A + c];
    if (lane == 0) {
      s.misc[r * 4 + 0] = a.logp[i];
      s.misc[r * 4 + 1] = (float)(((double)a.adv[i] - mean) / denom);
      s.misc[r * 4 + 2] = a.ret[i];
    }
  }
  if (a.stage) stage_wait();
  __syncthreads();
  // ---- forward with caches (mlp_forward nn.hpp:63-85) ----
  mlp_forward_tile_p(a.actor, lpa, s.x, ldx, s.aa, s.lda, nrows);
  mlp_forward_tile_p(a.critic, lpc, s.x, ldx, s.ca, s.ldc, nrows);
  // ---- per-row losses and head gradients (ppo.hpp:128-167) ----
  const float inv_n = 1.0f / (float)a.mb;
  const float* log_std = a.params + a.log_std_off;
  float* meanb = s.aa[a.actor.nl - 1];
  const int ldm = s.lda[a.actor.nl - 1];
  const int Q = (A + 3) / 4;
  int L = 1;
  while (L < Q && L < 32) L <<= 1;
  const int rpp = blockDim.x / L;
  const int lir = threadIdx.x % L;
  const int rmax = ((nrows + rpp - 1) / rpp) * rpp;
  for (int r = threadIdx.x / L; r < rmax; r += rpp) {
    const bool on = r < nrows;
    float lp = 0.0f;
    if (on)
      for (int d = lir; d < A; d += L) {
        const float ls = log_std[d];
        const float z = (s.actn[r * ldA + d] - meanb[r * ldm + d]) * expf(-ls);  // (a - mu) / sigma
        lp += (-0.5f * kLogTwoPiF - ls) - 0.5f * z * z;
      }
    for (int o = L / 2; o > 0; o >>= 1) lp += __shfl_xor_sync(0xffffffffu, lp, o, L);
    if (on) {
      const float ratio = expf(lp - s.misc[r * 4 + 0]);
      const float adv = s.misc[r * 4 + 1];
      const float surr1 = ratio * adv;
      const float lo = (float)(1.0 - a.clip), hi = (float)(1.0 + a.clip);
      const float clipped = (ratio < lo) ? lo : ((hi < ratio) ? hi : ratio);  // std::clamp
      const float surr2 = clipped * adv;
      const float dl_dlp = (surr1 <= surr2) ? -adv * ratio * inv_n : 0.0f;  // ppo.hpp:146
      for (int d = lir; d < A; d += L) {
        const float ls = log_std[d];
        const float isig = expf(-ls);
        const float z = (s.actn[r * ldA + d] - meanb[r * ldm + d]) * isig;
        meanb[r * ldm + d] = dl_dlp * (z * isig);  // dmean = dL/dlp * z / sigma, in place
        s.tmp[r * ldA + d] = dl_dlp * (z * z - 1.0f);
      }
      if (lir == 0) {
        s.loss[r * 2 + 0] = -((surr2 < surr1) ? surr2 : surr1) * inv_n;  // std::min (NaN-propagating)
        float* vb = s.ca[a.critic.nl - 1];
        const float err = vb[r * s.ldc[a.critic.nl - 1]] - s.misc[r * 4 + 2];
        s.loss[r * 2 + 1] = err * err * inv_n;
        vb[r * s.ldc[a.critic.nl - 1]] = (float)a.vf * 2.0f * err * inv_n;  // dV, in place
      }
    }
  }
  __syncthreads();
  float* part = a.partial + (size_t)blockIdx.x * a.Pext;
  const int ldp = a.ldw > ldA ? a.ldw : ldA;
  // ---- backward (mlp_backward_accumulate nn.hpp:105-132) ----
  for (int net = 0; net < 2; ++net) {
    const MlpDesc& d = net ? a.critic : a.actor;
    const LayerPtrs& lp = net ? lpc : lpa;
    float* const* acts = net ? s.ca : s.aa;
    const int* lds = net ? s.ldc : s.lda;
    const float* delta = acts[d.nl - 1];
    int ldd = lds[d.nl - 1];
    for (int l = d.nl - 1; l >= 0; --l) {
      const int in = d.dims[l], out = d.dims[l + 1];
      const float* lin = (l == 0) ? s.x : acts[l - 1];
      const int ldi = (l == 0) ? ldx : lds[l - 1];
      grad_w_tile(lin, ldi, in, delta, ldd, out, nrows, part + d.off[l]);
      if (l > 0) {
        float* dp = (delta == s.d0) ? s.d1 : s.d0;
        delta_prev_tile(delta, ldd, out, lp.W[l], lp.ldw[l], in, lin, ldi, dp, ldp, nrows);
        __syncthreads();
        delta = dp;
        ldd = ldp;
      }
    }
    __syncthreads();
  }
  // log_std partial (entropy term added once in the reduce) and loss sums
  for (int dd = threadIdx.x; dd < A; dd += blockDim.x) {
    float acc = 0.0f;
    for (int r = 0; r < nrows; ++r) acc += s.tmp[r * ldA + dd];
    part[a.log_std_off + dd] = acc;
  }
  if (threadIdx.x < 2) {
    float acc = 0.0f;
    for (int r = 0; r < nrows; ++r) acc += s.loss[r * 2 + threadIdx.x];
    part[a.P + threadIdx.x] = acc;
  }
}

struct ReduceArgs {
  const float* partial;
  int nparts, P, Pext, log_std_off, A;
  double ent;
  const float* params;
  float* grads;
  int32_t* status;    // [0] code, [1] detail
  int32_t* scratch;   // [0] ticket, [1] grad-nonfinite flag
  int64_t* t;         // Adam t (advanced when the step is accepted)
  int64_t* step;      // minibatch counter
  double* stats;      // sums: policy, value, entropy, count
  int apply;          // 0 = grads only (prb_ppo_loss_grads)
};

// Block = 32 parameters x 8 slices of the CTA partials; slice s sums partials
// s, s+8, ... with 4 independent accumulators, then the 8 slices are combined
// in a fixed order through shared memory: deterministic, and ~1,000 blocks of
// independent loads instead of one 128-long dependent chain per parameter.
constexpr int kRedCols = 32, kRedSlices = 8;

__global__ void __launch_bounds__(kRedCols * kRedSlices) ppo_reduce_kernel(ReduceArgs r) {
  if (r.status[0] != 0) return;
  __shared__ float part_sum[kRedSlices][kRedCols];
  const int col = threadIdx.x % kRedCols, slice = threadIdx.x / kRedCols;
  const int p = blockIdx.x * kRedCols + col;
  if (p < r.P) {
    float s0 = 0.f, s1 = 0.f, s2 = 0.f, s3 = 0.f;
    int b = slice;
    for (; b + 3 * kRedSlices < r.nparts; b += 4 * kRedSlices) {
      s0 += r.partial[(size_t)(b + 0 * kRedSlices) * r.Pext + p];
      s1 += r.partial[(size_t)(b + 1 * kRedSlices) * r.Pext + p];
      s2 += r.partial[(size_t)(b + 2 * kRedSlices) * r.Pext + p];
      s3 += r.partial[(size_t)(b + 3 * kRedSlices) * r.Pext + p];
    }
    for (; b < r.nparts; b += kRedSlices) s0 += r.partial[(size_t)b * r.Pext + p];
    part_sum[slice][col] = (s0 + s1) + (s2 + s3);
  }
  __syncthreads();
  int bad = 0;
  if (slice == 0 && p < r.P) {
    float acc = part_sum[0][col];
#pragma unroll
    for (int sl = 1; sl < kRedSlices; ++sl) acc += part_sum[sl][col];
    if (p >= r.log_std_off && p < r.log_std_off + r.A) acc -= (float)r.ent;  // ppo.hpp:157
    r.grads[p] = acc;
    bad = !isfinite(acc);
  }
  if (bad) atomicOr(&r.scratch[1], 1);
  __threadfence();
  __shared__ int last;
  if (threadIdx.x == 0) last = (atomicAdd(&r.scratch[0], 1) == (int)gridDim.x - 1);
  __syncthreads();
  if (!last || threadIdx.x != 0) return;
  __threadfence();
  double pl = 0.0, vl = 0.0;
  for (int b = 0; b < r.nparts; ++b) {
    pl += r.partial[(size_t)b * r.Pext + r.P];
    vl += r.partial[(size_t)b * r.Pext + r.P + 1];
  }
  double ent = 0.0;  // policy_entropy nn.hpp:273-277
  for (int d = 0; d < r.A; ++d) ent += 0.5 * (1.8378770664093454836 + 1.0) + (double)r.params[r.log_std_off + d];
  const int gbad = atomicAdd(&r.scratch[1], 0);
  r.scratch[0] = 0;
  r.scratch[1] = 0;
  if (!isfinite(pl)) {
    r.status[0] = PRB_ERR_NUMERIC;
    r.status[1] = 10;
  } else if (!isfinite(vl)) {
    r.status[0] = PRB_ERR_NUMERIC;
    r.status[1] = 11;
  } else if (!isfinite(ent)) {
    r.status[0] = PRB_ERR_NUMERIC;
    r.status[1] = 12;
  } else if (gbad && r.apply) {
    r.status[0] = PRB_ERR_NUMERIC;
    r.status[1] = 1;
  } else {
    r.stats[0] += pl;
    r.stats[1] += vl;
    r.stats[2] += ent;
    r.stats[3] += 1.0;
    if (r.apply) *r.t += 1;
  }
  *r.step += 1;
}

struct PpoWorkspace {
  DevBuf<float> partial;
  DevBuf<int32_t> scratch;
  DevBuf<int64_t> step;
  DevBuf<double> stats;
  DevBuf<uint32_t> perm;
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
  p.stage = 1;
  if (carve(p, nullptr, nullptr) > kSmemBudget) p.stage = 0;  // wide nets: weights stay in L2
  while (p.R > 8 && carve(p, nullptr, nullptr) > kSmemBudget) p.R /= 2;
  PRB_REQUIRE(carve(p, nullptr, nullptr) <= kSmemBudget, PRB_ERR_CONFIG, "ppo: network too wide for the SIMT tile");
  const int grid = (mb + p.R - 1) / p.R;
  if (ws.partial.n < (size_t)grid * p.Pext) ws.partial.alloc((size_t)grid * p.Pext);
  if (!ws.scratch.p) ws.scratch.alloc(4);
  if (!ws.step.p) ws.step.alloc(1);
  if (!ws.stats.p) ws.stats.alloc(4);
  p.partial = ws.partial.p;
  p.step = ws.step.p;
  return p;
}

void launch_step(const PpoArgs& p, prb_agent a, PpoWorkspace& ws, double ent, int apply, cudaStream_t s) {
  const int grid = (p.mb + p.R - 1) / p.R;
  const size_t smem = carve(p, nullptr, nullptr);
  ppo_fwd_bwd_kernel<<<grid, kPpoThreads, smem, s>>>(p);  // steps run inside CUDA graphs: no event scopes
  ReduceArgs r;
  r.partial = ws.partial.p;
  r.nparts = grid;
  r.P = p.P;
  r.Pext = p.Pext;
  r.log_std_off = p.log_std_off;
  r.A = p.A;
  r.ent = ent;
  r.params = p.params;
  r.grads = a->d_grads.p;
  r.status = a->d_status.p;
  r.scratch = ws.scratch.p;
  r.t = a->d_t.p;
  r.step = ws.step.p;
  r.stats = ws.stats.p;
  r.apply = apply;
  const int rgrid = (p.P + kRedCols - 1) / kRedCols;
  ppo_reduce_kernel<<<rgrid, kRedCols * kRedSlices, 0, s>>>(r);
  if (apply) prb_adam_launch(a, a->d_grads.p, a->d_status.p, s);
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

void set_smem_attr() {
  static bool done = false;
  if (!done) {
    PRB_CUDA(cudaFuncSetAttribute(ppo_fwd_bwd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemBudget));
    done = true;
  }
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
    if (src != dst) {
      int rc = prb_agent_copy(dst, src);
      if (rc) fail(rc, prb_last_error());
    }
    dst->lr = cfg->learning_rate;  // ppo.hpp:265
    PRB_CUDA(cudaMemsetAsync(dst->d_status.p, 0, 4 * sizeof(int32_t), s));
    prb_gae_launch(r->ctx, r->d_rew.p, r->d_val.p, r->d_done.p, r->d_boot.p, r->N, r->H, cfg->gamma, cfg->gae_lambda,
                   r->d_adv.p, r->d_ret.p, r->d_advstat.p, 1);
    if (r->ctx->stream != s) r->ctx->sync();
    r->gae_valid = true;
    r->normalized = true;
    PpoWorkspace ws;
    const int mb = (int)cfg->minibatch_size;
    PpoArgs p = make_args(dst, r, cfg, seed, ws, mb);
    const size_t steps = (size_t)cfg->epochs_per_update * p.nmb;
    if (perm) {
      std::vector<uint32_t> dev = ref_rows_to_device(r, perm, (size_t)cfg->epochs_per_update * n);
      ws.perm.alloc(dev.size());
      PRB_CUDA(cudaMemcpyAsync(ws.perm.p, dev.data(), dev.size() * sizeof(uint32_t), cudaMemcpyHostToDevice, s));
      p.perm = ws.perm.p;
      dst->ctx->sync();
    }
    PRB_CUDA(cudaMemsetAsync(ws.scratch.p, 0, 4 * sizeof(int32_t), s));
    PRB_CUDA(cudaMemsetAsync(ws.step.p, 0, sizeof(int64_t), s));
    PRB_CUDA(cudaMemsetAsync(ws.stats.p, 0, 4 * sizeof(double), s));
    // Minibatch steps are identical launches (the counter is on device):
    // capture a block of them once as a CUDA graph and replay it.
    const size_t kGraphSteps = 32;
    if (steps >= kGraphSteps) {
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
  });
}

int prb_ppo_loss_grads(prb_agent a, prb_rollout r, const uint64_t* rows, size_t n, const prb_ppo_config* cfg,
                       double* grads, double* losses) {
  return guard([&] {
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
    PRB_CUDA(cudaMemsetAsync(ws.scratch.p, 0, 4 * sizeof(int32_t), s));
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
      PRB_CUDA(cudaMemset(a->d_status.p, 0, 4 * sizeof(int32_t)));
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
